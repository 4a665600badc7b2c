#!/bin/bash
# A/B of runtime knobs (environment variables) on one box, bench lines interleaved.
# usage: VARS="base:_=0 a:FSCAN_X=1,FSCAN_Y=2" [REPS=2] [BARGS="--config 5"] bash tools/env_ab.sh
REPS=${REPS:-2}
BARGS=${BARGS:-}
for i in $(seq 1 $REPS); do
for v in $VARS; do
name=${v%%:*}; envs=$(echo "${v#*:}" | tr ',' ' ')
env $envs python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --no-proxy --no-exhaustive \
  --no-odometry --no-small $BARGS > gpurun_out/env_$name$i.json 2>gpurun_out/env_$name$i.err
python -c "import json;d=json.load(open('gpurun_out/env_$name$i.json'));print('$name', round(d['value']), d['bad_pairs'], d['clocks']['sm_mhz'], {k:round(x,2) for k,x in d['hbm_pipeline']['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/env_$name$i.err
done; done
