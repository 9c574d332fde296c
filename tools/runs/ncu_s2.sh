cd $GRAFT_REPO_ROOT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02s2_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pageable --extra-configs "" > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 600 ncu --kernel-name regex:normalize_rows_chunked --launch-skip 1 --launch-count 1 --set full --clock-control none --import-source on -o gpurun_out/k1_chunked_c4 python tools/time_normalize.py --configs c4 --reps 2 > gpurun_out/ncu_k1.log 2>&1; echo k1 rc=$?
timeout 600 ncu --kernel-name regex:normalize_rows_smem --launch-skip 1 --launch-count 1 --set full --clock-control none -o gpurun_out/k1_staged_c2 python tools/time_normalize.py --configs c2 --reps 2 > gpurun_out/ncu_k1b.log 2>&1; echo k1b rc=$?
timeout 900 python tools/time_ranks.py --configs c2,c3,c4,c5 --ps 1,2,4,8 --reps 3 > gpurun_out/ranks_s2.log 2>&1; echo ranks rc=$?
timeout 900 python tools/time_ranks.py --configs c2,c4 --ps 1,2,4,8 --reps 3 --method split >> gpurun_out/ranks_s2.log 2>&1; echo ranks2 rc=$?
