python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -c 1500 gpurun_out/bench3.json
