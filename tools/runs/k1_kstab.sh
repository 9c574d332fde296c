cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
for rep in 1 2; do ./tools/k1c_probe 32768 8192 | grep "ch=2048"; done
for k in 4 5 6; do echo "== CTAS=$k"; for rep in 1 2 3; do PCC_K1_CHUNK_CTAS=$k timeout 120 python tools/time_normalize.py --configs c4 --reps 5 | grep normalize; done; done
