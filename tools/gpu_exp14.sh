mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grad.py -x -q -p no:cacheprovider > gpurun_out/exp14_tests.log 2>&1
python tools/microbench.py --which acc > gpurun_out/exp14_acc.log 2>&1
python -c "
import sys, json, types, torch; sys.path.insert(0, '.')
import bench
a = types.SimpleNamespace(steps=10)
print(json.dumps(bench.bench_accumulate(torch.device('cuda:0'), a, bench.LLAMA8B_PARAMS)))" > gpurun_out/exp14_acc_full.log 2>&1
tail -2 gpurun_out/exp14_tests.log; cat gpurun_out/exp14_acc.log gpurun_out/exp14_acc_full.log
