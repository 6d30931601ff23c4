mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/exp4_tests.log 2>&1
for P in 2 4 8; do python tools/k4_run.py $P; done > gpurun_out/exp4_k4.log 2>&1
python tools/microbench.py --which acc > gpurun_out/exp4_acc.log 2>&1
./paper_2605_00539_b200/build/dropin_bench oracle/_ref/libagq_ref.so > gpurun_out/exp4_dropin.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_reduce128_pipe --launch-skip 2 --launch-count 1 -o gpurun_out/exp4_k4p8 python tools/k4_run.py 8 > gpurun_out/exp4_ncu.log 2>&1
tail -5 gpurun_out/exp4_tests.log; cat gpurun_out/exp4_k4.log gpurun_out/exp4_acc.log gpurun_out/exp4_dropin.log; tail -2 gpurun_out/exp4_ncu.log
