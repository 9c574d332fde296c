cd $GRAFT_REPO_ROOT
echo "== auto"; timeout 300 python tools/time_normalize.py --check --configs c2,c4,c5
timeout 300 python tools/time_normalize_split.py --configs c2,c4,c5
for k in 4 5 6 8 10 12; do echo "== CTAS=$k"; PCC_K1_CHUNK=1 PCC_K1_CHUNK_CTAS=$k timeout 300 python tools/time_normalize.py --configs c2,c4,c5 | grep normalize; done
echo "== chunk off"; PCC_K1_CHUNK=0 timeout 300 python tools/time_normalize.py --configs c2,c4 | grep normalize
PCC_K1_CHUNK=1 timeout 900 python -m pytest tests -m gpu -x -q -k "normal or split or fused or k1 or parity or bcast or exchange or golden" 2>&1 | tail -3
