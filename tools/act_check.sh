python -m pytest tests -m gpu -q -x --tb=short 2>&1 | tail -3
python tools/microbench.py --which act 2>&1 | grep quant
python bench.py --steps 20 --warmup 5 --no-e2e --no-accumulate --no-allreduce --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('value', j['value'], j['roofline'], j['c1'])"
