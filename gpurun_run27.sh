CMD="python bench.py --pairs 256 --steps 2 --warmup 3 --no-e2e --no-cpu --no-exhaustive --no-odometry"
$CMD > gpurun_out/small27.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"xlat_cols|xlat_rows|xlat_out|rot_cols|rot_rows" -s 5 -c 5 -o gpurun_out/prof27 $CMD > gpurun_out/ncu27.log 2>&1
echo ncu rc=$?
