python -m pytest tests -m gpu -q 2>&1 | tail -3
bash tools/profile_pack.sh r01b
for c in 2 3 5; do python bench.py --config $c --steps 10 --warmup 3 --no-e2e > gpurun_out/r01b_bench_c$c.json 2>/dev/null; echo "c$c rc=$?"; done
python -c "
import json
d=json.load(open('gpurun_out/r01b_bench.json'))
print(d['value'], d['e2e'], d.get('exhaustive_search'), d['cpu_baseline'], d['roofline']['frac'])
print(d['hbm_pipeline'])
"
