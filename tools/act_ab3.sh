# same-box A/B/C of the act kernels: default vs two variants
for rep in 1 2; do for v in default $1 $2; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  python bench.py --steps 20 --warmup 5 --no-e2e --no-accumulate --no-allreduce --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print('$v', 'value', j['value'], 'quant', r['achieved'] if r['kernel']=='k_quant_warp' else r.get('k_quant_warp_GBs'), 'dequant', r.get('k_dequant_warp_GBs', r['achieved']), 'c1_us', j['c1']['us_per_roundtrip'])"
done; done
