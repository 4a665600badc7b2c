VARS="G H I" bash gpurun_ab.sh
