#!/bin/bash
# tools/sweep.sh "config4 config3" "4:16 4:8 2:8 4:4"   (look:chunk pairs)
for c in $1; do for lc in $2; do
  export HB_LOOK_ROUNDS=${lc%%:*} HB_CHUNK_ROUNDS=${lc##*:}
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/sw.json 2> gpurun_out/sw.err
  python -c "import json;d=json.load(open('gpurun_out/sw.json'));r=d['roofline'];print('$c look=$HB_LOOK_ROUNDS chunk=$HB_CHUNK_ROUNDS', round(d['ms_per_step'],3),'ms', round(r['frac'],3))" || tail -2 gpurun_out/sw.err
done; done
