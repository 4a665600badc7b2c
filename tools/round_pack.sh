#!/bin/bash
# Round measurement pack (ONE GPU): both bench arms (default command lines), the
# other configs' lines, the ncu launch list of a C4 step and one --set full
# capture of a production chunk. Outputs gpurun_out/<tag>_*. usage: bash tools/round_pack.sh r02
set -u
T=${1:-r02}
O=gpurun_out
python bench.py --impl reference > $O/${T}_ref.json 2> $O/${T}_ref.err; echo "ref rc=$?"
python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
for c in 1 2 3 5; do
  python bench.py --config $c --steps 20 --warmup 5 --no-cpu --no-exhaustive --no-odometry > $O/${T}_c$c.json 2> $O/${T}_c$c.err
  echo "c$c rc=$?"
done
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-proxy --no-exhaustive --no-odometry --no-small"
$CMD > $O/${T}_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(rot_|xlat_|finalize)" -c 600 --csv --log-file $O/${T}_launches.csv $CMD > $O/${T}_ncu_list.log 2>&1
echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"rot_rows|rot_cols|rot_gather|rot_polar|xlat_rows|xlat_cols|xlat_out|finalize" -s 18 -c 9 -o $O/${T}_full $CMD > $O/${T}_ncu_full.log 2>&1
echo "ncu full rc=$?"
