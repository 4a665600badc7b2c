python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tests/gpu_probe.py 2>&1 | grep -E "cfg(2|4|5) pair" | head -6
VARS="G H" bash gpurun_ab.sh
