mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_cpp_dropin.py tests/test_multigpu.py -x -q -p no:cacheprovider > gpurun_out/exp11_tests.log 2>&1
python -c "
import sys, json, types, torch; sys.path.insert(0, '.')
import bench
print(json.dumps(bench.bench_c1(torch.device('cuda:0'), types.SimpleNamespace(steps=20))))" > gpurun_out/exp11_c1.log 2>&1
tail -3 gpurun_out/exp11_tests.log; cat gpurun_out/exp11_c1.log
