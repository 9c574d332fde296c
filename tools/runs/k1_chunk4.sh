cd $GRAFT_REPO_ROOT
for k in 1 2 3; do echo "== chunk4 CTAS=$k"; PCC_K1_CHUNK=1 PCC_K1_CHUNK_CTAS=$k timeout 300 python tools/time_normalize.py --check --configs c2,c4,c5 | grep -E "normalize|False"; PCC_K1_CHUNK=1 PCC_K1_CHUNK_CTAS=$k timeout 300 python tools/time_normalize_split.py --configs c2,c4,c5; done
echo "== chunk4 auto"; timeout 300 python tools/time_normalize.py --configs c2,c4,c5 | grep normalize
echo "== chunk1 (old)"; PCC_K1_CHUNK4=0 timeout 300 python tools/time_normalize.py --configs c4 | grep normalize; PCC_K1_CHUNK4=0 timeout 300 python tools/time_normalize_split.py --configs c4
PCC_K1_CHUNK=1 timeout 900 python -m pytest tests -m gpu -x -q -k "normal or split or fused or k1 or parity or bcast or exchange or golden" 2>&1 | tail -2
