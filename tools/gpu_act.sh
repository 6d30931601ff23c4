# activation codec check: GPU codec tests + the C2/C1 bench sub-lines (no e2e/CPU legs)
TAG=${1:-act}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_grouped.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
tail -2 gpurun_out/${TAG}_tests.log
for i in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-accumulate > gpurun_out/${TAG}_bench$i.log 2>&1
python - <<PY
import json
for l in open("gpurun_out/${TAG}_bench$i.log"):
    if l.startswith("{"):
        d = json.loads(l)
        print("value", d["value"], "roofline", d["roofline"]["achieved"], d["roofline"]["frac"])
        print("c2_stage", json.dumps(d.get("c2_stage"))[:400])
        print("c1", json.dumps(d.get("c1"))[:600])
PY
done
