for i in 1 2; do for v in 0 2 1; do
FSCAN_PDL=$v python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-proxy --no-exhaustive --no-odometry > gpurun_out/pdl_$v$i.json 2> gpurun_out/pdl_$v$i.err
python -c "import json;d=json.load(open('gpurun_out/pdl_$v$i.json'));s=d['small_batches'];print('PDL$v', round(d['value']), d['bad_pairs'], 'c1 us', s['c1']['us_per_call_median'], 'c2', round(s['c2']['value']), s['c2']['us_per_call_median'])" || tail -3 gpurun_out/pdl_$v$i.err
done; done
for v in 0 2; do FSCAN_PDL=$v python bench.py --config 5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-proxy --no-exhaustive --no-odometry --no-small > gpurun_out/pdl5_$v.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/pdl5_$v.json'));print('C5 PDL$v', round(d['value']))"; done
