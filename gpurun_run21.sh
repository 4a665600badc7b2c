VARS="M2 P" bash gpurun_ab.sh
