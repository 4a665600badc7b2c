python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench7.json 2> gpurun_out/bench7.err; python -c "import json;d=json.load(open('gpurun_out/bench7.json'));print(d['value'], d['hbm_pipeline']['kernel_ms_per_step'])"
