#!/bin/bash
# C2 (64 pairs of 256^2) pairs/s over lane counts (chunk = ceil(64 / lanes)); FSCAN_PDL as given (default rule)
for rep in 1 2; do
for cfg in "3 1" "2 1" "4 1" "6 1" "8 1" "3 0" "3 2"; do
  set -- $cfg
  env FSCAN_LANES=$1 FSCAN_PDL=$2 python bench.py --config 2 --steps 50 --warmup 5 --no-e2e --no-cpu --no-proxy --no-exhaustive --no-odometry > gpurun_out/c2s_$1_$2_$rep.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/c2s_$1_$2_$rep.json'));print('C2 lanes $1 pdl $2', round(d['value']))"
done; done
