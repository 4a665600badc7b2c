#!/bin/bash
# C5 pairs/s over lane counts / chunk sizes (FSCAN_LANES / FSCAN_CHUNK), interleaved
for rep in 1 2; do
for cfg in "3 0" "4 0" "2 0" "3 32" "4 32" "3 48"; do
  set -- $cfg
  if [ "$2" = "0" ]; then CH=""; else CH="FSCAN_CHUNK=$2"; fi
  env FSCAN_LANES=$1 $CH python bench.py --config 5 --steps 10 --warmup 3 --no-e2e --no-cpu --no-proxy --no-exhaustive --no-odometry --no-small > gpurun_out/c5s_$1_$2_$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c5s_$1_$2_$rep.json'));print('C5 lanes $1 chunk $2', round(d['value']))"
done; done
