cd $GRAFT_REPO_ROOT
timeout 300 python tools/time_normalize.py --check --configs c1,c2,c3,c4,c5
timeout 300 python tools/time_normalize_split.py --configs c2,c3,c4,c5
timeout 900 python -m pytest tests -m gpu -x -q -k "normal or split or fused or k1 or parity or bcast or exchange or golden" 2>&1 | tail -4
