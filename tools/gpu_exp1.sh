mkdir -p gpurun_out
python tools/ab_act.py $PWD/paper_2605_00539_b200/libagq_cuda.so $PWD/paper_2605_00539_b200/build/seg8/libagq_cuda.so > gpurun_out/exp1_ab_seg.log 2>&1
python -c "
import sys, json, torch; sys.path.insert(0,'.')
import bench
print(json.dumps(bench.bench_dropin(torch.device('cuda:0'))))" > gpurun_out/exp1_dropin.log 2>&1
python tools/k4_run.py 8 > gpurun_out/exp1_k4.log 2>&1
python tools/k4_run.py 2 >> gpurun_out/exp1_k4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_reduce128_pipe --launch-skip 2 --launch-count 1 -o gpurun_out/exp1_k4p8 python tools/k4_run.py 8 > gpurun_out/exp1_ncu.log 2>&1
tail -5 gpurun_out/exp1_ab_seg.log; cat gpurun_out/exp1_dropin.log gpurun_out/exp1_k4.log; tail -3 gpurun_out/exp1_ncu.log
