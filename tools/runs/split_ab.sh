cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do for mc in 0 1; do echo "== rep $rep PCC_SPLIT_MC=$mc"; PCC_SPLIT_MC=$mc timeout 200 python tools/split_check.py --config c4 --reps 3 --skip-dmma --sustain 5 | grep -E "syrk|sustain|clock|MHz"; done; done
