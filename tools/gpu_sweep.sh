# C5 sweep at N GPUs. usage: bash tools/gpu_sweep.sh N TAG
N=$1; TAG=$2
mkdir -p gpurun_out
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus $N --sweep > gpurun_out/${TAG}_sweep.log 2>&1
python - <<PY
import json
for l in open("gpurun_out/${TAG}_sweep.log"):
    if l.startswith("{"):
        for r in json.loads(l)["sweep"]:
            print(r["case"], {k: v for k, v in r.items() if k.endswith("_us") or k == "speedup_vs_bf16"})
PY
