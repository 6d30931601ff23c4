# fused all-reduce: 2 (default) vs 3 CTAs/SM launch bounds, N GPUs
N=${1:-4}
for rep in 1 2; do for v in default p2pmb3; do
  if [ $v = default ]; then unset AGQ_LIB; unset AGQ_P2P_CTAS_PER_SM; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; export AGQ_P2P_CTAS_PER_SM=3; fi
  timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29720+rep)) bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-accumulate --algos p2p 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', json.dumps(d['allreduce']['p2p']))"
done; done
