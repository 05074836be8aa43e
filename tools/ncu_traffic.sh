#!/bin/bash
# DRAM bytes per dense step of each config's union kernels (profiles/ncu_traffic.json) and
# the launch list of the bench workload.  Run on the GPU box; writes gpurun_out/ncu_*.csv.
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in ${1:-config2 config3 config4 config5}; do
  timeout 900 ncu --metrics $M --clock-control none -k regex:"k_light|k_heavy" --csv \
    --log-file gpurun_out/ncu_traffic_$c.csv python bench.py --config $c --steps 1 --warmup 3 \
    --no-e2e --no-cpu-baseline --no-per-config > gpurun_out/ncu_traffic_$c.log 2>&1 || tail -3 gpurun_out/ncu_traffic_$c.log
done
if [ -z "$2" ]; then
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/ncu_launches_config4.csv \
  python bench.py --steps 5 --warmup 3 --e2e-steps 1 --e2e-warmup 0 --no-cpu-baseline --no-per-config \
  --no-e2e-int64 > gpurun_out/ncu_launches_config4.log 2>&1 || tail -3 gpurun_out/ncu_launches_config4.log
fi
