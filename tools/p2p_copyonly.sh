# fused all-reduce vs the same kernel with compute removed (transfer bound)
for mode in normal copy; do
  if [ $mode = copy ]; then export AGQ_P2P_COPYONLY=1; fi
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$1 --master-addr=127.0.0.1 --master-port=2955$1 bench.py --gpus $1 --steps 3 --warmup 3 --no-e2e --no-accumulate --algos p2p 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$mode', json.dumps(d['allreduce']['p2p']))" >> gpurun_out/p2p_copyonly.log
done
