# 2-GPU check of the error-word change: multi-GPU tests + C5 sweep.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -x -q -p no:cacheprovider > gpurun_out/errw_mp_tests.log 2>&1
tail -3 gpurun_out/errw_mp_tests.log
bash tools/gpu_sweep.sh 2 errw2 | head -6
