set -x
cd $GRAFT_REPO_ROOT
for k in 0 1; do for ow in 4 6; do
  echo "== PCC_K1_STREAM=$k OW=$ow"
  PCC_K1_STREAM=$k PCC_K1S_OW=$ow timeout 300 python tools/time_normalize.py --check --configs c2,c4,c5
  PCC_K1_STREAM=$k PCC_K1S_OW=$ow timeout 300 python tools/time_normalize_split.py --configs c2,c4,c5
done; done
PCC_K1_STREAM=1 timeout 900 python -m pytest tests -m gpu -x -q -k "normal or split or fused or k1 or parity" 2>&1 | tail -5
