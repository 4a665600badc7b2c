set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -c 2500 gpurun_out/bench2.json
CMD="python bench.py --pairs 512 --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:xlat_cols -s 2 -c 1 -o gpurun_out/prof_xlat_cols $CMD > gpurun_out/ncu2.log 2>&1
echo ncu rc=$?
tail -3 gpurun_out/ncu2.log
