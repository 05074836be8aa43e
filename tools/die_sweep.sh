#!/bin/bash
# usage: tools/die_sweep.sh "<env assignments>;<env assignments>;..." [config] [steps]
# die-affine heavy items: dense step of config 5 under env overrides (HB_DIE, HB_DIE_HINT_MB,
# HB_L2_PERSIST_MB, HB_PERSIST_WINDOW, HB_HINT_MB)
IFS=';' read -ra V <<< "$1"
c=${2:-config5}
for v in "${V[@]}"; do
  env $v timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-per-config --steps ${3:-10} > gpurun_out/ds.json 2> gpurun_out/ds.err
  python -c "import json;d=json.load(open('gpurun_out/ds.json'));r=d['roofline'];print('$v $c', round(d['ms_per_step'],3),'ms', round(r['frac'],3))" || tail -2 gpurun_out/ds.err
done
