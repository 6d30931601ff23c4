# One GPU box pass: the GPU test suite, smoke, one bench line of each arm.
# usage (inside gpurun): bash tools/gpu_check.sh TAG
TAG=${1:-check}
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/${TAG}_smi.log 2>&1
nproc >> gpurun_out/${TAG}_smi.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/${TAG}_gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_n1.log 2>&1
echo "bench rc=$?" >> gpurun_out/${TAG}_bench_n1.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref_n1.log 2>&1
tail -3 gpurun_out/${TAG}_gpu_tests.log; tail -2 gpurun_out/${TAG}_smoke.log; tail -c 3000 gpurun_out/${TAG}_bench_n1.log
