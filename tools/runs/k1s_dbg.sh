cd $GRAFT_REPO_ROOT
PCC_K1_STREAM=1 timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "normalize_bit_exact_vs_reference_golden" 2>&1 | grep -E "Error|assert|case|name" | head -20
PCC_K1_STREAM=1 timeout 600 ncu --kernel-name regex:normalize_rows_stream --launch-skip 1 --launch-count 1 --set full --clock-control none -o gpurun_out/k1s_c4 python tools/time_normalize.py --configs c4 --reps 1 > gpurun_out/k1s_ncu.log 2>&1
tail -3 gpurun_out/k1s_ncu.log
