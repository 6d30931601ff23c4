# same-box A/B of the act step: default vs environment "$1=$2"
for rep in 1 2; do for v in default alt; do
  if [ $v = default ]; then unset $1; else export $1=$2; fi
  python bench.py --steps 20 --warmup 5 --no-e2e --no-accumulate --no-allreduce --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); r=j['roofline']; print('$v' if '$v'=='default' else '$1=$2', 'value', j['value'], 'quant', r['achieved'] if r['kernel']=='k_quant_warp' else r.get('k_quant_warp_GBs'), 'dequant', r.get('k_dequant_warp_GBs', r['achieved']), 'c1_us', j['c1']['us_per_roundtrip'])"
done; done
unset $1
