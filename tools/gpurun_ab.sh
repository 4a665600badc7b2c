#!/bin/bash
# A/B: alternate builds of the library (tools/ab_build.sh -> ab/libNAME.so) on the
# same box, C4 bench lines interleaved. usage: VARS="A B" [BARGS=...] bash tools/gpurun_ab.sh
VARS=${VARS:-"A B"}
REPS=${REPS:-2}
for i in $(seq 1 $REPS); do
for v in $VARS; do
FSCAN_LIB=$PWD/ab/lib$v.so python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-proxy --no-exhaustive \
  --no-odometry --no-small $BARGS > gpurun_out/ab_$v$i.json 2>gpurun_out/ab_$v$i.err
python -c "import json;d=json.load(open('gpurun_out/ab_$v$i.json'));print('$v', round(d['value']), d['bad_pairs'], {k:round(x,2) for k,x in d['hbm_pipeline']['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/ab_$v$i.err
done; done
