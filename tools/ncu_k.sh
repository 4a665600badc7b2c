#!/bin/bash
# ncu --set full of one kernel family for several A/B builds: usage
#   KRE=xlat_cols VARS="V1 R112" TAG=r02e bash tools/ncu_k.sh
set -u
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-proxy --no-exhaustive --no-odometry"
for v in $VARS; do
  if [ "$v" = "default" ]; then L=""; else L="FSCAN_LIB=$PWD/ab/lib$v.so"; fi
  env $L ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s ${SKIP:-4} -c ${COUNT:-2} \
    -o gpurun_out/${TAG}_$v $CMD > gpurun_out/${TAG}_$v.log 2>&1
  echo "$v ncu rc=$?"
done
