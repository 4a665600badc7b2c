python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tests/gpu_probe.py 2>&1 | grep -E "cfg(2|4|5) pair" | head -6
python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/b17.json 2>gpurun_out/b17.err; python -c "import json;d=json.load(open('gpurun_out/b17.json'));print(d['value'], d['hbm_pipeline']['kernel_ms_per_step'])"
CMD="python bench.py --pairs 256 --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rot_rows|rot_cols|rot_gather|rot_polar|xlat_rows|xlat_out|xlat_cols" -s 7 -c 7 -o gpurun_out/prof17 $CMD > gpurun_out/ncu17.log 2>&1
echo ncu rc=$?
