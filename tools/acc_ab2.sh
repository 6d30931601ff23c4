# K3 A/B (default vs variant $1): 2^28 microbench + C3 (8.03e9 params) in the bench
V=${1:-prev}
for rep in 1 2; do for v in default $V; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  echo "== $v"; python tools/microbench.py --which acc 2>&1 | grep case
  python bench.py --steps 3 --warmup 3 --no-e2e --no-allreduce --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; j=json.loads(sys.stdin.read()); print('C3', j['accumulate']['ms'], j['accumulate']['GBs'])"
done; done
