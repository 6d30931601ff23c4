# A/B of whole bench C2 step lines between library builds: bash tools/ab_bench.sh libA libB ...
for rnd in 1 2 3; do
  for lib in "$@"; do
    AGQ_LIB=$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-accumulate --no-allreduce 2>/dev/null | python -c "
import json, sys
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); r = d['roofline']
        print('$rnd', '$lib', d['value'], d['ms_per_step'], r['achieved'], r.get('k_dequant_warp_GBs'), d['c2_stage']['b4']['ms'], d['c2_stage']['b8']['ms'], d['c1']['us_per_roundtrip'], flush=True)
"
  done
done
