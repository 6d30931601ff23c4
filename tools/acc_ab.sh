python -m pytest tests -m gpu -x -q -k "grad or smoke or numerics" 2>&1 | tail -2
for v in default tab0; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  echo "== $v"; python tools/microbench.py --which acc 2>&1 | grep case
  python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3', j['accumulate'])"
done
