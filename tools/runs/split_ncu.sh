cd $GRAFT_REPO_ROOT
timeout 600 ncu --kernel-name regex:syrk_split --launch-skip 1 --launch-count 1 --set full --clock-control none -o gpurun_out/split_c2 python tools/split_check.py --config c2 --reps 2 --skip-dmma > gpurun_out/split_ncu.log 2>&1
tail -2 gpurun_out/split_ncu.log
