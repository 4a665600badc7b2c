python -m pytest tests -m gpu -q 2>&1 | tail -2
bash tools/profile_pack.sh r01c
for c in 2 3 5; do python bench.py --config $c --steps 10 --warmup 3 --no-e2e > gpurun_out/r01c_bench_c$c.json 2>/dev/null; echo "c$c rc=$?"; done
python -c "
import json
d=json.load(open('gpurun_out/r01c_bench.json'))
print(d['value'], d['e2e'], d.get('exhaustive_search'), d.get('odometry_chain'), d['cpu_baseline'], d['roofline'])
print(d['hbm_pipeline'])
"
