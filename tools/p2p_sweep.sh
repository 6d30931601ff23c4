for c in 1 2 4 8; do
  AGQ_P2P_CTAS_PER_SM=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=2953$c bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e --no-accumulate --algos p2p --ar-elements 2147483648 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('ctas/sm=$c', json.dumps(d['allreduce']['p2p']), 'bf16', d['allreduce']['bf16_nccl'])" >> gpurun_out/p2p_sweep.log
done
