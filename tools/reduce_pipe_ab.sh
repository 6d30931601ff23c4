# A/B of K4: cp.async ring (2/3/4 stages) vs the direct-load kernel. Parity first.
python -m pytest tests/test_gpu_grad.py -x -q --tb=short 2>&1 | tail -3
for r in 1 2; do
for v in direct 2 3 4; do
  if [ $v = direct ]; then export AGQ_RED_PIPE=0; else unset AGQ_RED_PIPE; export AGQ_RED_STAGES=$v; fi
  echo "== $v"; python tools/microbench.py --which reduce 2>&1 | grep case
done
done
