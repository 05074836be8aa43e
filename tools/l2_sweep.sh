#!/bin/bash
# config 5 dense step vs the L2 head size (HB_HINT_MB evict_last range, HB_L2_PERSIST_MB window)
cd $GRAFT_REPO_ROOT
for hm in $1; do for pm in $2; do
HB_HINT_MB=$hm HB_L2_PERSIST_MB=$pm timeout 300 python bench.py --config ${3:-config5} --no-cpu-baseline --no-e2e --no-per-config --steps 10 > gpurun_out/l2.json 2> gpurun_out/l2.err
python -c "import json;d=json.load(open('gpurun_out/l2.json'));print('hint $hm persist $pm', round(d['ms_per_step'],3),'ms', round(d['roofline']['frac'],3))" || tail -2 gpurun_out/l2.err
done; done
