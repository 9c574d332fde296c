cd $GRAFT_REPO_ROOT
./tools/k1c_probe 32768 8192 | grep "ch=2048"; ./tools/k1c_probe 16384 4096 | grep "ch=2048"
for c in 0 1; do echo "== PCC_K1_CHUNK=$c"; PCC_K1_CHUNK=$c timeout 300 python tools/time_normalize.py --check --configs c1,c2,c3,c4,c5; PCC_K1_CHUNK=$c timeout 300 python tools/time_normalize_split.py --configs c2,c3,c4,c5; done
for k in 6 8; do echo "== CTAS=$k"; PCC_K1_CHUNK=1 PCC_K1_CHUNK_CTAS=$k timeout 300 python tools/time_normalize.py --configs c2,c4,c5 | grep normalize; PCC_K1_CHUNK=1 PCC_K1_CHUNK_CTAS=$k timeout 300 python tools/time_normalize_split.py --configs c2,c4,c5; done
for c in 0 1; do PCC_K1_CHUNK=$c timeout 900 python -m pytest tests -m gpu -x -q -k "normal or split or fused or k1 or parity or bcast or exchange or golden" 2>&1 | tail -2; done
