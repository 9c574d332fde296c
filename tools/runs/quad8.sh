cd $GRAFT_REPO_ROOT
for q in 0 1; do echo "== PCC_QUAD8=$q"; PCC_QUAD8=$q timeout 600 python tools/time_ranks.py --configs c3,c1,c2 --ps 1,2,4,8 --reps 5; done
PCC_QUAD8=1 timeout 900 python -m pytest tests -m gpu -x -q -k "quad or tail or parity or range or invariance or workers" 2>&1 | tail -3
