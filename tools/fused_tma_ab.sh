# fused all-reduce: per-thread pulls (default) vs TMA-pipelined pulls (AGQ_P2P_TMA=1)
N=${1:-2}
AGQ_P2P_TMA=1 timeout 400 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29701 tests/mp_allreduce_check.py 2>&1 | grep -E "failures|MISMATCH|Error|error" | head -5
for rep in 1 2; do for v in default tma; do
  if [ $v = tma ]; then export AGQ_P2P_TMA=1; else unset AGQ_P2P_TMA; fi
  timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29710+rep)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-accumulate --algos p2p 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', json.dumps(d['allreduce']['p2p']))"
done; done
