# push all-reduce: two kernels (default) vs one overlapped kernel (AGQ_PUSH_OVERLAP=1)
N=${1:-2}
AGQ_PUSH_OVERLAP=1 timeout 400 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29941 tests/mp_allreduce_check.py 2>&1 | grep -E "failures|MISMATCH|rror" | head -5
for rep in 1 2; do for v in default overlap; do
  if [ $v = overlap ]; then export AGQ_PUSH_OVERLAP=1; else unset AGQ_PUSH_OVERLAP; fi
  timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29950+rep)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-accumulate --algos p2p,push 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); a=d['allreduce']; print('$v', 'p2p', a['p2p']['ms'], 'push', a['push']['ms'], a.get('push_equals_nccl'), 'bf16', a['bf16_nccl']['ms'])"
done; done
unset AGQ_PUSH_OVERLAP
