set -x
nvidia-smi -L
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/final_gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final_bench_n1.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_bench_ref_n1.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29701 bench.py --gpus 2 > gpurun_out/final_bench_n2.log 2>&1
tail -2 gpurun_out/final_gpu_tests.log; tail -1 gpurun_out/final_smoke.log
