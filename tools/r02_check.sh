#!/bin/bash
# gpu tests + both bench arms (default command lines), outputs under gpurun_out/<tag>_*
set -u
OUT=gpurun_out
T=${1:-r02b}
python -m pytest tests -m gpu -x -q ${PYTEST_K:-} > $OUT/${T}_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 $OUT/${T}_gputest.log
python bench.py --impl reference > $OUT/${T}_ref.json 2> $OUT/${T}_ref.err; echo "ref rc=$?"
python bench.py > $OUT/${T}_bench.json 2> $OUT/${T}_bench.err; echo "bench rc=$?"
