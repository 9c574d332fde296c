cd $GRAFT_REPO_ROOT
for e in 0 1 9 17; do echo "== probe EXP $e"; for s in "16384 4096" "32768 8192" "65536 2048"; do ./tools/k1s2_probe_e$e $s; done; done
for k in 1; do for ow in 4; do
  echo "== PCC_K1_STREAM=$k OW=$ow"
  PCC_K1_STREAM=$k PCC_K1S_OW=$ow timeout 300 python tools/time_normalize.py --check --configs c2,c4,c5
  PCC_K1_STREAM=$k PCC_K1S_OW=$ow timeout 300 python tools/time_normalize_split.py --configs c2,c4,c5
done; done
PCC_K1_STREAM=1 timeout 900 python -m pytest tests -m gpu -x -q -k "normal or split or fused or k1 or parity or bcast or exchange" 2>&1 | tail -5
