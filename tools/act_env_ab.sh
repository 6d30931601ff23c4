# same-box A/B of the act kernels: default vs AGQ_ACT_KERNEL=$1 (+ its codec tests)
K=${1:-cpa}
AGQ_ACT_KERNEL=$K python -m pytest tests/test_gpu_codec.py -q -x 2>&1 | tail -1
for rep in 1 2; do for v in default $K; do
  if [ $v = default ]; then unset AGQ_ACT_KERNEL; else export AGQ_ACT_KERNEL=$v; fi
  python bench.py --steps 20 --warmup 5 --no-e2e --no-accumulate --no-allreduce --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print('$v', 'value', j['value'], 'quant', r['achieved'] if r['kernel']=='k_quant_warp' else r.get('k_quant_warp_GBs'), 'dequant', r.get('k_dequant_warp_GBs', r['achieved']), 'c1_us', j['c1']['us_per_roundtrip'])"
done; done
unset AGQ_ACT_KERNEL
