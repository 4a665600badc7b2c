python -m pytest tests -m gpu -x -q 2>&1 | tail -2
FSCAN_CHUNK=128 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b10.json 2>gpurun_out/b10.err; python -c "import json;d=json.load(open('gpurun_out/b10.json'));print(d['value'], d['hbm_pipeline']['kernel_ms_per_step'])"
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b10b.json 2>gpurun_out/b10b.err; python -c "import json;d=json.load(open('gpurun_out/b10b.json'));print(d['value'], d['hbm_pipeline']['kernel_ms_per_step'])"
