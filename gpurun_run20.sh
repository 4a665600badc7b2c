CMD="python bench.py --pairs 256 --steps 2 --warmup 3 --no-e2e --no-cpu"
for v in G I; do
FSCAN_LIB=$PWD/ab/lib$v.so $CMD > /dev/null 2>&1
FSCAN_LIB=$PWD/ab/lib$v.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,smsp__inst_executed.sum --clock-control none -k regex:"rot_rows" -s 2 -c 2 --csv $CMD > gpurun_out/ncu20_$v.csv 2>gpurun_out/ncu20_$v.err
done
echo done
