python tests/gpu_probe.py 2>&1 | tail -30
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -c 1200 gpurun_out/bench4.json; tail -3 gpurun_out/bench4.err
