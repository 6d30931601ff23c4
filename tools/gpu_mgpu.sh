# multi-GPU evidence on N GPUs: tests, bench C4
# with forced-algorithm BF16 baselines. usage: bash tools/gpu_mgpu.sh N TAG
N=$1; TAG=$2
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -x -q -p no:cacheprovider > gpurun_out/${TAG}_mp_tests.log 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29622 bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1
tail -3 gpurun_out/${TAG}_mp_tests.log; python - <<PY
import json
for l in open("gpurun_out/${TAG}_bench.log"):
    if l.startswith("{"):
        d = json.loads(l); print(json.dumps(d.get("allreduce"), indent=1)); print("value", d["value"])
PY
