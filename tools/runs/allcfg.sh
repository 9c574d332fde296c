cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_s2.jsonl 2> gpurun_out/ref_s2.err; echo ref rc=$?; tail -c 400 gpurun_out/ref_s2.jsonl
for c in c1 c2 c3 c5; do
  st=10; [ $c = c1 ] && st=50
  timeout 900 python bench.py --config $c --steps $st --warmup 3 --extra-configs "" --cpu-fraction 0.0625 >> gpurun_out/allcfg_s2.jsonl 2>> gpurun_out/allcfg_s2.err; echo $c rc=$?
done
