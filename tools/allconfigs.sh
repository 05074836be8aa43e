#!/bin/bash
# usage: tools/allconfigs.sh [configs]   -- dense step + e2e per config
for c in ${1:-config1 config2 config3 config4 config5s config5}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 30 > gpurun_out/all_$c.json 2> gpurun_out/all_$c.err
  python - "$c" <<'PY' || tail -3 gpurun_out/all_$1.err
import json, sys
c = sys.argv[1]
d = json.load(open(f"gpurun_out/all_{c}.json"))
r, e = d["roofline"], d["e2e"]
print(c, d["config"]["schedule"], f"step {d['ms_per_step']:.4f} ms", f"alg {r['achieved']:.0f} GB/s",
      f"frac {r['frac']:.3f}", f"e2e {e['seconds_per_run']:.4f} s/run {e['iterations']} it",
      f"{e['value']:.3e}")
PY
done
