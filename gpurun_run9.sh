python -m pytest tests -m gpu -x -q -k "chunking or c4 or golden" 2>&1 | tail -2
for L in 2 4; do for C in 32 128 512; do
FSCAN_LANES=$L FSCAN_CHUNK=$C python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b9.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/b9.json'));print('lanes $L chunk $C', d['value'], d['ms_per_step'])"
done; done
