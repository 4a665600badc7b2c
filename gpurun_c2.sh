for i in 1 2 3; do for v in A B; do
echo $v $(FSCAN_LIB=$PWD/ab/lib$v.so python bench.py --config 2 --steps 30 --warmup 5 --no-e2e --no-cpu --no-exhaustive --no-odometry | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['hbm_pipeline']['kernel_ms_per_step'])")
done; done
for v in A B; do echo $v $(FSCAN_LIB=$PWD/ab/lib$v.so python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-exhaustive --no-odometry | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']))"); done
