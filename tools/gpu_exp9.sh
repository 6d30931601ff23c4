mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grad.py tests/test_gpu_codec.py tests/test_multigpu.py -x -q -p no:cacheprovider > gpurun_out/exp9_tests.log 2>&1
for P in 2 4 8; do python tools/k4_run.py $P; done > gpurun_out/exp9_k4.log 2>&1
python tools/microbench.py --which acc > gpurun_out/exp9_acc.log 2>&1
tail -3 gpurun_out/exp9_tests.log; cat gpurun_out/exp9_k4.log gpurun_out/exp9_acc.log
