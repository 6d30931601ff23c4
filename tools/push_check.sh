# push all-reduce: bit-exact multi-rank check, then C4 timing of all three algorithms
N=${1:-2}
timeout 400 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29801 tests/mp_allreduce_check.py 2>&1 | grep -v "^\*\|NCCL version" | tail -5
for rep in 1 2; do
timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29810+rep)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-accumulate 2>&1 | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps(d['allreduce']))"
done
