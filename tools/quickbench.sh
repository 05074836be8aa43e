#!/bin/bash
# usage: tools/quickbench.sh "config4 config3" [steps]
for c in $1; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${2:-30} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d['roofline'];print('$c', round(d['ms_per_step'],3),'ms', round(r['achieved']),'GB/s', round(r['frac'],3), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/bench_$c.err
done
