mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/exp7_topo.log 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -x -q -p no:cacheprovider > gpurun_out/exp7_mp_tests.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/nvlink_bytes.py > gpurun_out/exp7_nvlink_bytes.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/exp7_bench_n2.log 2>&1
NCCL_ALGO=NVLS NCCL_DEBUG=INFO timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-accumulate --algos p2p > gpurun_out/exp7_bench_n2_nvls.log 2> gpurun_out/exp7_bench_n2_nvls.err
grep -E "NVLS|nvls" gpurun_out/exp7_bench_n2_nvls.err | head -5 > gpurun_out/exp7_nvls_info.log
tail -3 gpurun_out/exp7_mp_tests.log; cat gpurun_out/exp7_nvlink_bytes.log; tail -c 2500 gpurun_out/exp7_bench_n2.log; tail -c 1500 gpurun_out/exp7_bench_n2_nvls.log; cat gpurun_out/exp7_nvls_info.log
