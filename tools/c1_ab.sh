# C1 (4096^2, b=4) per-kernel times, default build vs a variant
V=${1:-prev}
for rep in 1 2; do for v in default $V; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  echo "== $v"; python tools/microbench.py --which act --n 16777216 --bits 4 --iters 200 2>&1 | grep case
done; done
