#!/bin/bash
# C4 pairs/s for lane counts / chunk sizes (FSCAN_LANES / FSCAN_CHUNK), interleaved
for rep in 1 2; do
for cfg in "3 0" "2 0" "4 0" "3 96" "3 64" "4 96"; do
  set -- $cfg
  if [ "$2" = "0" ]; then CH=""; else CH="FSCAN_CHUNK=$2"; fi
  env FSCAN_LANES=$1 $CH python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-proxy --no-exhaustive --no-odometry --no-small > gpurun_out/lanes_$1_$2_$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/lanes_$1_$2_$rep.json'));print('lanes $1 chunk $2', round(d['value']))"
done; done
