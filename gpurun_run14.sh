python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tests/gpu_probe.py 2>&1 | grep -E "cfg(4|5) pair" | head -4
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b14.json 2>gpurun_out/b14.err; python -c "import json;d=json.load(open('gpurun_out/b14.json'));print(d['value'], d['hbm_pipeline']['kernel_ms_per_step'])"
