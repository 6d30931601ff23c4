# push all-reduce: fused reduce+gather (default) vs AGQ_PUSH_SPLIT=1, N GPUs
N=${1:-4}
AGQ_PUSH_SPLIT=1 timeout 400 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29901 tests/mp_allreduce_check.py 2>&1 | grep failures
for rep in 1 2; do for v in default split; do
  if [ $v = split ]; then export AGQ_PUSH_SPLIT=1; else unset AGQ_PUSH_SPLIT; fi
  timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29910+rep)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-accumulate --algos push 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', json.dumps(d['allreduce']['push']))"
done; done
