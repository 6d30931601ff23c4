# A/B of the K4 decode: block table (default) vs full 256-entry table (red0)
python -m pytest tests -m gpu -x -q --tb=short 2>&1 | tail -4
for v in default red0 redmb3 redmb4; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  echo "== $v"; python tools/microbench.py --which reduce 2>&1 | grep case
done
