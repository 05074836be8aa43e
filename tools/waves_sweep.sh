#!/bin/bash
# usage: tools/waves_sweep.sh "config4 config3" "0 1 2 3" [tickets 0|1] [steps]
#   HB_GRID_WAVES sweep of the light kernel's grid (0 = the old 8-CTA-per-SM cap), with the
#   chunk tickets on (default) or off (HB_TICKETS=0: grid-stride chunks)
for w in $2; do
  for c in $1; do
    HB_TICKETS=${3:-1} HB_GRID_WAVES=$w timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-per-config --steps ${4:-30} > gpurun_out/wv.json 2> gpurun_out/wv.err
    python -c "import json;d=json.load(open('gpurun_out/wv.json'));r=d['roofline'];print('tickets=${3:-1} waves=$w $c', round(d['ms_per_step'],4),'ms', round(r['frac'],3))" || tail -2 gpurun_out/wv.err
  done
done
