#!/bin/bash
# e2e + dense step of one config under each schedule order
cd $GRAFT_REPO_ROOT
for sc in ${2:-identity window}; do
timeout 300 python bench.py --config ${1:-config3} --schedule $sc --no-cpu-baseline --no-per-config --no-e2e-int64 --steps 30 --e2e-steps 5 > gpurun_out/s.json 2> gpurun_out/s.err
python -c "import json;d=json.load(open('gpurun_out/s.json'));e=d['e2e'];print('${1:-config3} $sc', round(d['ms_per_step'],3),'ms', 'e2e', round(e['seconds_per_run']*1000,2),'ms', e['iterations'],'it')" || tail -2 gpurun_out/s.err
done
