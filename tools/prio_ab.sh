for rep in 1 2 3 4; do for v in 0 1; do
FSCAN_LANE_PRIO=$v python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-proxy --no-exhaustive --no-odometry --no-small > gpurun_out/prio_$v$rep.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/prio_$v$rep.json'));print('PRIO$v', round(d['value']), d['clocks']['sm_mhz'])"
done; done
