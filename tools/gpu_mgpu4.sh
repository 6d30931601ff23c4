# 4-GPU evidence: real-rank tests, bench C4 with forced-algorithm BF16
# baselines, the C5 sweep. usage: bash tools/gpu_mgpu4.sh TAG
TAG=$1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_multigpu.py -x -q -p no:cacheprovider > gpurun_out/${TAG}_mp_tests.log 2>&1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --bf16-algos NVLS,NVLSTree,Ring,Tree > gpurun_out/${TAG}_bench.log 2>&1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 4 --sweep > gpurun_out/${TAG}_sweep.log 2>&1
tail -3 gpurun_out/${TAG}_mp_tests.log; python - <<PY
import json
for f in ("gpurun_out/${TAG}_bench.log", "gpurun_out/${TAG}_sweep.log"):
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            if "allreduce" in d: print(json.dumps(d["allreduce"], indent=1)); print("value", d["value"])
            if "sweep" in d:
                for r in d["sweep"]: print(r["case"], r.get("p2p_us"), r.get("bf16_nccl_us"), r.get("speedup_vs_bf16"))
PY
