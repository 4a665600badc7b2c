set -u
for v in $VARS; do
  if [ "$v" != BASE ]; then
  FSCAN_LIB=$PWD/ab/lib$v.so python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "baseline_configs or golden or two_pass" > gpurun_out/ab_test_$v.log 2>&1; echo "$v test rc=$?"; tail -2 gpurun_out/ab_test_$v.log
  fi
done
bash tools/gpurun_ab.sh
