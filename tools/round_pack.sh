#!/bin/bash
# Full measurement pack for the round's profiles/ refresh (run under gpurun on
# ONE GPU): tools/profile_pack.sh (C4 bench line, launch list, full ncu capture)
# plus the other configs' bench lines. usage: bash tools/round_pack.sh <tag>
TAG=${1:-r01}
bash tools/profile_pack.sh $TAG
for c in 2 3 5; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/${TAG}_c$c.json 2> gpurun_out/${TAG}_c$c.err
  echo "c$c rc=$?"
done
