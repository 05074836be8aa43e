#!/bin/bash
# config 5 dense step with the packed hot head on / off, per library variant
cd $GRAFT_REPO_ROOT
cp paper_1308_2144_b200/libhyperball_b200.so /tmp/k.so
for v in $1; do
  cp sweep/lib_$v.so paper_1308_2144_b200/libhyperball_b200.so
  for hp in ${2:-1 0}; do
    HB_HOT_PACK=$hp timeout 300 python bench.py --config config5 --no-cpu-baseline --no-e2e --no-per-config --steps 10 > gpurun_out/sw.json 2> gpurun_out/sw.err
    python -c "import json;d=json.load(open('gpurun_out/sw.json'));r=d['roofline'];print('$v hot=$hp config5', round(d['ms_per_step'],3),'ms', round(r['frac'],3))" || tail -2 gpurun_out/sw.err
  done
done
cp /tmp/k.so paper_1308_2144_b200/libhyperball_b200.so
