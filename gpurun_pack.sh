bash tools/profile_pack.sh r01d
for c in 2 3 5; do python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r01d_c$c.json 2> gpurun_out/r01d_c$c.err; echo "c$c rc=$?"; done
