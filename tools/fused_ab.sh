# Fused all-reduce: bit-exact multi-rank check (EPT 16 and 8), then C4 timing
# with the block-table decode (default) vs the full table (red0). Arg: N GPUs.
N=${1:-2}
timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29601 tests/mp_allreduce_check.py 2>&1 | tail -3
AGQ_P2P_EPT=8 timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29602 tests/mp_allreduce_check.py 2>&1 | tail -3
port=29610
for v in default red0 default red0; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  port=$((port+1))
  timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-accumulate --algos p2p 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', json.dumps(d['allreduce']))"
done
