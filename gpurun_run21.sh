VARS="G M" bash gpurun_ab.sh
