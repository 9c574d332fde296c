cd $GRAFT_REPO_ROOT
for c in c1 c3 c2 c4; do for mc in 0 1; do echo "== $c PCC_SPLIT_MC=$mc"; PCC_SPLIT_MC=$mc timeout 120 python tools/split_check.py --config $c --reps 5 --hash --skip-dmma; done; done
PCC_SPLIT_MC=1 timeout 600 python -m pytest tests/test_gpu_split.py -x -q 2>&1 | tail -4
