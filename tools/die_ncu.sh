#!/bin/bash
# k_heavy_partial of config 5's dense step, with and without die-affine items: time, DRAM
# bytes, L2 hit rate, fabric sectors, issue activity (gpurun_out/die_ncu_<tag>.csv)
cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_ltcfabric.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for tag in ${1:-die nodie}; do
  v="HB_DIE=1"; [ $tag = nodie ] && v="HB_DIE=0"
  env $v ${2:-} timeout 900 ncu --metrics $M --clock-control none -k regex:"k_heavy_partial|k_light|k_heavy_finish" -s 9 -c 4 --csv \
    --log-file gpurun_out/die_ncu_$tag.csv python bench.py --config ${CFG:-config5} --steps 1 --warmup 3 \
    --no-e2e --no-cpu-baseline --no-per-config > gpurun_out/die_ncu_$tag.log 2>&1 || tail -3 gpurun_out/die_ncu_$tag.log
done
