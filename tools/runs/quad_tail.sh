cd $GRAFT_REPO_ROOT
for r in 1 2 0; do echo "== PCC_QUAD_TAIL_ROUNDS=$r"; PCC_QUAD_TAIL_ROUNDS=$r timeout 600 python tools/time_ranks.py --configs c3,c2 --ps 1,2,4,8 --reps 5; done
