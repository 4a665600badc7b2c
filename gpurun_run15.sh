python -m pytest tests -m gpu -x -q 2>&1 | tail -2
CMD="python bench.py --pairs 256 --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rot_rows|rot_cols|rot_gather|rot_polar|xlat_rows|xlat_out|xlat_cols" -s 7 -c 7 -o gpurun_out/prof15 $CMD > gpurun_out/ncu15.log 2>&1
echo ncu rc=$?
