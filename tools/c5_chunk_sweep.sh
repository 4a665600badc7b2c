for rep in 1 2; do for ch in 0 48 63; do
  if [ "$ch" = "0" ]; then E=""; else E="FSCAN_CHUNK=$ch"; fi
  env $E python bench.py --config 5 --steps 10 --warmup 3 --no-e2e --no-cpu --no-proxy --no-exhaustive --no-odometry --no-small > gpurun_out/c5ch_$ch_$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c5ch_$ch_$rep.json'));print('chunk $ch', round(d['value']), {k:round(x,2) for k,x in d['hbm_pipeline']['kernel_ms_per_step'].items()})"
done; done
