set -x
python -m pytest tests -m gpu -x -q -k "grad or numerics or smoke" 2>&1 | tail -3
for v in m0 default m8888 mEEEE mFFFF; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  echo "== $v"; python tools/microbench.py --which acc 2>&1 | tail -4; python tools/microbench.py --which reduce 2>&1 | tail -8
done
