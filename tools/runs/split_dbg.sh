cd $GRAFT_REPO_ROOT
for d in 0 1 2 6; do echo "== PCC_SPLIT_DEBUG=$d (mc off)"; PCC_SPLIT_MC=0 PCC_SPLIT_DEBUG=$d timeout 120 python tools/split_check.py --config c2 --reps 5 --skip-dmma | grep syrk; done
echo "== mc on"; timeout 120 python tools/split_check.py --config c2 --reps 5 --skip-dmma | grep syrk
