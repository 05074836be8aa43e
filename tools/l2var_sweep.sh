#!/bin/bash
# usage: tools/l2var_sweep.sh "variants" "persist MBs" [config]
cd $GRAFT_REPO_ROOT
cp paper_1308_2144_b200/libhyperball_b200.so /tmp/lib_keep.so
for v in $1; do
  cp sweep/lib_$v.so paper_1308_2144_b200/libhyperball_b200.so
  for pm in $2; do
    HB_L2_PERSIST_MB=$pm timeout 300 python bench.py --config ${3:-config5} --no-cpu-baseline --no-e2e --no-per-config --steps 10 > gpurun_out/l2.json 2> gpurun_out/l2.err
    python -c "import json;d=json.load(open('gpurun_out/l2.json'));print('$v persist $pm', round(d['ms_per_step'],3),'ms', round(d['roofline']['frac'],3))" || tail -2 gpurun_out/l2.err
  done
done
cp /tmp/lib_keep.so paper_1308_2144_b200/libhyperball_b200.so
