#!/bin/bash
# usage: tools/libsweep2.sh "config3:identity config3:window" "base A B" [steps]
cp paper_1308_2144_b200/libhyperball_b200.so /tmp/lib_keep.so
for v in $2; do
  cp sweep/lib_$v.so paper_1308_2144_b200/libhyperball_b200.so
  for cs in $1; do
    c=${cs%%:*}; sc=${cs##*:}
    timeout 300 python bench.py --config $c --schedule $sc --no-cpu-baseline --no-e2e --steps ${3:-30} > gpurun_out/sw.json 2> gpurun_out/sw.err
    python -c "import json;d=json.load(open('gpurun_out/sw.json'));r=d['roofline'];print('$v $c $sc', round(d['ms_per_step'],4),'ms', round(r['frac'],3))" || tail -2 gpurun_out/sw.err
  done
done
cp /tmp/lib_keep.so paper_1308_2144_b200/libhyperball_b200.so
