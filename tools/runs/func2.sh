cd $GRAFT_REPO_ROOT
for ex in local p2p; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --config c4 --u-exchange $ex --no-exact --no-pageable --extra-configs "" 2>gpurun_out/func2_$ex.err | tail -1 > gpurun_out/func2_$ex.jsonl; echo "$ex rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/func2_$ex.jsonl').read())
print('$ex', d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['config'].get('u_exchange_e2e','')[:60], d['config'].get('world_size'), d.get('split_mode',{}).get('ms_per_step'))
"
done
