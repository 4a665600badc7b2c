python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 2 3 5; do python bench.py --config $c --steps 10 --warmup 3 --no-e2e > gpurun_out/b11_c$c.json 2>gpurun_out/b11_c$c.err; python -c "import json;d=json.load(open('gpurun_out/b11_c$c.json'));print($c, d['value'], d['ms_per_step'], d['cpu_baseline'], d['hbm_pipeline']['kernel_ms_per_step'])"; done
bash tools/profile_pack.sh r01b
python -c "import json;d=json.load(open('gpurun_out/r01b_bench.json'));print(d['value'], d['e2e'], d['cpu_baseline'], d['roofline'])"
