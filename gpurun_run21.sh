VARS="M O" bash gpurun_ab.sh
