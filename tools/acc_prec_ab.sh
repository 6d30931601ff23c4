# K3 rounded-precision A/B: default vs block-table decode / 2 CTAs per SM for PREC != 0
for rep in 1 2; do for v in default ${@:-tabprec minb2p tabminb2}; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  echo "== $v"; timeout 300 python tools/microbench.py --which acc 2>&1 | grep -E "case|errors"
done; done
