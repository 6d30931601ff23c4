# FP4 BF16-input quantizer occupancy A/B (default vs build/q4m2) + K3 rates of the default build
for rep in 1 2; do for v in default q4m2; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  echo "== $v"; timeout 300 python tools/codec_rates.py 2>&1 | grep -i "fp4\|e2m1"
done; done
unset AGQ_LIB
echo "== default acc"; timeout 300 python tools/microbench.py --which acc 2>&1 | grep -E "case|errors"
