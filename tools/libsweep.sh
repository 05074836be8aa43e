#!/bin/bash
# usage: tools/libsweep.sh "config3 config5s" "base A B" [steps]
#   swaps sweep/lib_<v>.so (variant builds, -D overrides) in and benches each config
cp paper_1308_2144_b200/libhyperball_b200.so /tmp/lib_keep.so
for v in $2; do
  cp sweep/lib_$v.so paper_1308_2144_b200/libhyperball_b200.so
  for c in $1; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --no-per-config --steps ${3:-30} > gpurun_out/sw.json 2> gpurun_out/sw.err
    python -c "import json;d=json.load(open('gpurun_out/sw.json'));r=d['roofline'];print('$v $c', round(d['ms_per_step'],3),'ms', round(r['frac'],3))" || tail -2 gpurun_out/sw.err
  done
done
cp /tmp/lib_keep.so paper_1308_2144_b200/libhyperball_b200.so
