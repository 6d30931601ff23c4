"""A/B of activation-kernel builds on one box: C1 round trip (quant+dequant,
16 rotating 4096^2 BF16 copies), C1 quant / dequant alone, and the C2 silu
tensor (235M) quant / dequant at b=4 and 8. usage:
  python tools/ab_act.py libA.so libB.so [...]   (alternates, 3 rounds)"""
import json
import os
import subprocess
import sys

CHILD = r'''
import json, os, sys, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_2605_00539_b200 as A
from paper_2605_00539_b200 import _lib as L
dev = torch.device("cuda:0")
sp = torch.cuda.current_stream().cuda_stream
def timeit(fn, iters):
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for i in range(iters): fn(i)
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us
res = {}
for n, R, tag in ((4096 * 4096, 16, "c1"), (16384 * 14336, 3, "c2silu")):
    xs = [torch.randn(n, device=dev).to(torch.bfloat16) for _ in range(R)]
    ys = [torch.empty_like(x) for x in xs]
    for b in ((4,) if tag == "c1" else (4, 8)):
        cs = [torch.empty(n * b // 8, dtype=torch.uint8, device=dev) for _ in range(R)]
        ss = [torch.empty(n // 128, dtype=torch.float32, device=dev) for _ in range(R)]
        q = lambda i: L.lib.agq_quantize(xs[i % R].data_ptr(), 1, n, b, 128, 0, cs[i % R].data_ptr(), 0, ss[i % R].data_ptr(), None, sp)
        d = lambda i: L.lib.agq_dequantize(cs[i % R].data_ptr(), 0, ss[i % R].data_ptr(), n, b, 128, 0, ys[i % R].data_ptr(), 1, 0, None, sp)
        it = 80 if tag == "c1" else 10
        res[f"{tag}_q{b}"] = timeit(q, it)
        res[f"{tag}_d{b}"] = timeit(d, it)
        if tag == "c1":
            res["c1_rt"] = timeit(lambda i: (q(i), d(i)), it)
    del xs, ys
    torch.cuda.empty_cache()
print(json.dumps({k: round(v, 2) for k, v in res.items()}))
'''

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = sys.argv[1:]
for rnd in range(3):
    for lib in libs:
        env = dict(os.environ, AGQ_LIB=lib, ROOT=root)
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        print(rnd, os.path.basename(os.path.dirname(lib)) or lib, r.stdout.strip() or r.stderr[-500:],
              flush=True)
