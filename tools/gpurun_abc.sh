# A/B over configs: VARS libs, CFGS configs
for c in ${CFGS:-2 4 5}; do for v in $VARS; do
FSCAN_LIB=$PWD/ab/lib$v.so python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu --no-exhaustive --no-odometry 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('C$c $v', d['value'], d['hbm_pipeline']['kernel_ms_per_step'].get('xlat_cols'))"
done; done
