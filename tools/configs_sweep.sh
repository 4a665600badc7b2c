#!/bin/bash
# bench lines of the other BASELINE configs (quick): gpurun_out/<tag>_c<id>.json
T=${1:-r02q}
for c in 1 2 3 5; do
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu --no-exhaustive --no-odometry > gpurun_out/${T}_c$c.json 2> gpurun_out/${T}_c$c.err
  python -c "import json;d=json.load(open('gpurun_out/${T}_c$c.json'));print('C$c', round(d['value']), d['step_ms'], {k:round(x,3) for k,x in d['hbm_pipeline']['kernel_ms_per_step'].items()})" || tail -3 gpurun_out/${T}_c$c.err
done
