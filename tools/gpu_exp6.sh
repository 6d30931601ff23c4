mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grad.py -x -q -p no:cacheprovider > gpurun_out/exp6_tests.log 2>&1
for P in 2 4 8; do python tools/k4_run.py $P; done > gpurun_out/exp6_k4.log 2>&1
python tools/microbench.py --which acc > gpurun_out/exp6_acc.log 2>&1
python tools/c1_run.py > gpurun_out/exp6_c1.log 2>&1
ncu --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_.*quant_warp --launch-skip 40 --launch-count 8 --csv python tools/c1_run.py 30 > gpurun_out/exp6_c1_ncu.csv 2>&1
tail -3 gpurun_out/exp6_tests.log; cat gpurun_out/exp6_k4.log gpurun_out/exp6_acc.log gpurun_out/exp6_c1.log; grep -E "gpu__time_duration" gpurun_out/exp6_c1_ncu.csv | head -8
