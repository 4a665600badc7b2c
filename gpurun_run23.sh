python -m pytest tests -m gpu -q -k "polar or c3 or baseline_configs" 2>&1 | tail -2
python bench.py --config 3 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/c3.json 2>gpurun_out/c3.err; python -c "
import json; d=json.load(open('gpurun_out/c3.json')); print(d['value'], d['hbm_pipeline']['kernel_ms_per_step'], d['roofline'])"
