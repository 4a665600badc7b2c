CMD="python bench.py --pairs 256 --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"xlat_rows|xlat_cols" -s 2 -c 2 -o gpurun_out/prof13 $CMD > gpurun_out/ncu13.log 2>&1
echo ncu rc=$?
