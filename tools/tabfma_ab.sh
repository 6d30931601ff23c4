# A/B of the block-table decode's accumulate: one FFMA2 onto acc (default)
# vs FMUL2 + FADD (nofma, the previous build). Parity first.
python -m pytest tests/test_gpu_grad.py tests/test_gpu_codec.py -x -q --tb=short 2>&1 | tail -3
for r in 1 2; do
for v in default nofma; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  echo "== $v"; python tools/microbench.py --which reduce 2>&1 | grep case
  python tools/microbench.py --which acc 2>&1 | grep case
done
done
