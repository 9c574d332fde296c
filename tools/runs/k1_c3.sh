cd $GRAFT_REPO_ROOT
timeout 600 ncu --kernel-name regex:normalize_rows --launch-skip 1 --launch-count 1 --set full --clock-control none -o gpurun_out/k1_c3 python tools/time_normalize.py --configs c3 --reps 2 > gpurun_out/ncu_k1c3.log 2>&1; echo rc=$?
for r in 1 2 3 4 5 6 7 8; do PCC_NORMALIZE_ROWS=$r timeout 120 python tools/time_normalize.py --configs c3 | grep normalize; done
for t in 64 128 256; do PCC_NORMALIZE_THREADS=$t timeout 120 python tools/time_normalize.py --configs c3 | grep normalize; done
