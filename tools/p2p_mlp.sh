# fused all-reduce at N GPUs: elements-per-thread x CTAs-per-SM grid
N=${1:-4}
port=29700
for ept in 16 8; do for c in 1 2 3 4; do
  port=$((port+1))
  r=$(AGQ_P2P_EPT=$ept AGQ_P2P_CTAS_PER_SM=$c timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-accumulate --algos p2p 2>/dev/null | grep '^{' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps(d['allreduce']['p2p']))")
  echo "ept=$ept ctas_per_sm=$c $r"
done; done
