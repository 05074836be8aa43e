#!/bin/bash
# Full ncu captures (one launch each, 4th dense step) of the dominant union kernels:
# gpurun_out/r2c_<config>_<kernel>.ncu-rep.  usage: tools/ncu_full.sh "config4:k_light config5:k_heavy_partial"
cd $GRAFT_REPO_ROOT
for ck in $1; do
  c=${ck%%:*}; k=${ck##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -s 3 -c 1 -f \
    -o gpurun_out/r2c_${c}_${k} python bench.py --config $c --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline --no-per-config > gpurun_out/ncu_full_${c}_${k}.log 2>&1 || tail -3 gpurun_out/ncu_full_${c}_${k}.log
done
