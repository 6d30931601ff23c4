# K3 BF16-local occupancy A/B: default (3 CTAs/SM) vs build/bl4 (4 CTAs/SM, 64 registers)
for rep in 1 2 3; do for v in default bl4; do
  if [ $v = default ]; then unset AGQ_LIB; else export AGQ_LIB=$PWD/paper_2605_00539_b200/build/$v/libagq_cuda.so; fi
  echo "== $v"; timeout 300 python tools/microbench.py --which acc 2>&1 | grep -E "case|errors"
done; done
