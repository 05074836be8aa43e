#!/bin/bash
# usage: tools/winmult_sweep.sh "config3:window config4:auto" "1 4 16"  -- HB_WINDOW_MULT sweep
for m in $2; do
  for cs in $1; do
    c=${cs%%:*}; sch=${cs##*:}
    HB_WINDOW_MULT=$m timeout 600 python bench.py --config $c --schedule $sch --no-cpu-baseline --no-per-config --steps ${3:-30} > gpurun_out/wm.json 2> gpurun_out/wm.err
    python -c "import json;d=json.load(open('gpurun_out/wm.json'));r=d['roofline'];e=d['e2e'];print('mult=$m $c $sch', round(d['ms_per_step'],4),'ms', round(r['frac'],3), 'e2e', round(e['seconds_per_run']*1e3,2),'ms')" || tail -2 gpurun_out/wm.err
  done
done
