# A/B: alternate builds of the library on the same box
VARS=${VARS:-"A B"}
for i in 1 2; do
for v in $VARS; do
FSCAN_LIB=$PWD/ab/lib$v.so python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu $BARGS > gpurun_out/ab_$v$i.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/ab_$v$i.json'));print('$v', round(d['value']), {k:round(x,2) for k,x in d['hbm_pipeline']['kernel_ms_per_step'].items()})"
done; done
