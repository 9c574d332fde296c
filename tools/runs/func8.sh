cd $GRAFT_REPO_ROOT
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 8 --steps 2 --warmup 3 --config c2 --no-exact --no-pageable --extra-configs "" 2>gpurun_out/func8.err | tail -1 > gpurun_out/func8.jsonl; echo "rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 8 --steps 2 --warmup 1 --config c2 2>gpurun_out/func8r.err | tail -1 > gpurun_out/func8r.jsonl; echo "ref rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/func8.jsonl').read())
print(d['n_gpus'], d['value'], d['ms_per_step'], d['e2e']['ms_per_step'], d['config'].get('world_size'), d['config'].get('k1_rows_per_rank'))
d=json.loads(open('gpurun_out/func8r.jsonl').read()); print(d.get('impl'), d.get('value'), d.get('unavailable'))
"
