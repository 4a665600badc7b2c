#!/bin/bash
# round-2 baseline pack: gpu tests, bench line, full ncu of one production-size C4 chunk
set -u
OUT=gpurun_out
T=${1:-r02a}
python -m pytest tests -m gpu -x -q > $OUT/${T}_gputest.log 2>&1; echo "gputest rc=$?"
python bench.py --steps 20 --warmup 5 > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-exhaustive --no-odometry"
ncu --set full --clock-control none --import-source on -k regex:"xlat_rows|xlat_cols|xlat_out|rot_rows|rot_cols|rot_gather" -s 12 -c 6 -o $OUT/${T}_full $CMD > $OUT/${T}_ncu_full.log 2>&1
echo "ncu rc=$?"
