mkdir -p gpurun_out
python tools/ab_act.py $PWD/paper_2605_00539_b200/libagq_cuda.so $PWD/paper_2605_00539_b200/build/seg32/libagq_cuda.so > gpurun_out/exp2_ab_seg.log 2>&1
./paper_2605_00539_b200/build/dropin_bench oracle/_ref/libagq_ref.so > gpurun_out/exp2_dropin.log 2>&1
./paper_2605_00539_b200/build/dropin_bench oracle/_ref/libagq_ref.so >> gpurun_out/exp2_dropin.log 2>&1
timeout 900 python -m pytest tests/test_gpu_grouped.py tests/test_cpp_dropin.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/exp2_tests.log 2>&1
cat gpurun_out/exp2_ab_seg.log gpurun_out/exp2_dropin.log; tail -5 gpurun_out/exp2_tests.log
