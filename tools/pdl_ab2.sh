for rep in 1 2; do for v in 0 1; do
FSCAN_PDL=$v python bench.py --config 5 --steps 10 --warmup 3 --no-cpu --no-e2e --no-proxy --no-exhaustive --no-odometry --no-small > gpurun_out/p5_$v$rep.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/p5_$v$rep.json'));print('C5 PDL$v', round(d['value']))"
FSCAN_PDL=$v python bench.py --config 1 --steps 200 --warmup 20 --no-cpu --no-e2e --no-proxy --no-exhaustive --no-odometry > gpurun_out/p1_$v$rep.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/p1_$v$rep.json'));print('C1 PDL$v', round(d['value']), d['step_ms'])"
done; done
