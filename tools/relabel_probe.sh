#!/bin/bash
# k_relabel* time and DRAM bytes on config 5's end-to-end run, per library variant
cd $GRAFT_REPO_ROOT
cp paper_1308_2144_b200/libhyperball_b200.so /tmp/lib_keep.so
for v in $1; do
  cp sweep/lib_$v.so paper_1308_2144_b200/libhyperball_b200.so
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_relabel|k_map_ids" --csv --log-file gpurun_out/relabel_$v.csv python bench.py --config ${2:-config5} --steps 1 --warmup 3 \
    --e2e-steps 1 --e2e-warmup 0 --no-e2e-int64 --no-per-config --no-cpu-baseline > gpurun_out/relabel_$v.log 2>&1 || tail -3 gpurun_out/relabel_$v.log
  python tools/launch_table.py gpurun_out/relabel_$v.csv | sed "s/^/$v /"
  timeout 600 python bench.py --config ${2:-config5} --steps 3 --warmup 3 --e2e-steps 3 --e2e-warmup 1 --no-e2e-int64 --no-per-config --no-cpu-baseline > gpurun_out/rl.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/rl.json'));print('$v e2e', round(d['e2e']['seconds_per_run'],4), 's')"
done
cp /tmp/lib_keep.so paper_1308_2144_b200/libhyperball_b200.so
