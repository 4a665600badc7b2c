#!/bin/bash
# Standard measurement pack for one round (run under gpurun on ONE GPU):
#   bench line (C4), launch list (ncu gpu__time_duration), full ncu capture of the
#   translation-stage kernels, all written to gpurun_out/<tag>_*.
# usage: bash tools/profile_pack.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out
python bench.py --steps 20 --warmup 5 > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?"
CMD="python bench.py --pairs 256 --steps 2 --warmup 3 --no-e2e --no-cpu --no-exhaustive --no-odometry"
$CMD > $OUT/${TAG}_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $OUT/${TAG}_launches.csv $CMD > $OUT/${TAG}_ncu_list.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rot_rows|rot_cols|rot_gather|rot_polar|xlat_rows|xlat_cols|xlat_out|finalize" -s 8 -c 8 -o $OUT/${TAG}_full $CMD > $OUT/${TAG}_ncu_full.log 2>&1
echo "ncu rc=$?"
