cd $GRAFT_REPO_ROOT
for c in config3 config2; do for sc in identity window degree; do
timeout 300 python bench.py --config $c --schedule $sc --no-cpu-baseline --no-e2e --no-per-config --steps 30 > gpurun_out/s.json 2> gpurun_out/s.err
python -c "import json;d=json.load(open('gpurun_out/s.json'));r=d['roofline'];print('$c $sc', round(d['ms_per_step'],3),'ms', round(r['frac'],3))" || tail -2 gpurun_out/s.err
done; done
