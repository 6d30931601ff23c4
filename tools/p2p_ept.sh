# fused all-reduce: parity + timing for both elements-per-thread variants
N=$1
for ept in 16 8; do
  AGQ_P2P_EPT=$ept timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=$((29500+ept)) tests/mp_allreduce_check.py 2>&1 | grep failures | sed "s/^/ept=$ept /" >> gpurun_out/p2p_ept.log
  AGQ_P2P_EPT=$ept timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=$((29600+ept)) bench.py --gpus $N --steps 3 --warmup 3 --no-e2e --no-accumulate --algos p2p 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ept=$ept', json.dumps(d['allreduce']['p2p']))" >> gpurun_out/p2p_ept.log
done
