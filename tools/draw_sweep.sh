#!/bin/bash
# usage: tools/draw_sweep.sh "config5 config5s" "dpw:dmax ..."  -- heavy-item ticket run length
for v in $2; do
  for c in $1; do
    HB_DRAWS_PER_WARP=${v%%:*} HB_DRAW_MAX=${v##*:} timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --no-per-config --steps ${3:-20} > gpurun_out/dr.json 2> gpurun_out/dr.err
    python -c "import json;d=json.load(open('gpurun_out/dr.json'));r=d['roofline'];print('draws=$v $c', round(d['ms_per_step'],4),'ms', round(r['frac'],3))" || tail -2 gpurun_out/dr.err
  done
done
