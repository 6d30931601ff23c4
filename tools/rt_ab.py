"""A/B of the fused round-trip kernel builds: C1 fused round trip us."""
import os, subprocess, sys
CHILD = r'''
import os, sys, torch
sys.path.insert(0, os.environ["ROOT"])
import paper_2605_00539_b200 as A
from paper_2605_00539_b200 import _lib as L
n, R = 4096 * 4096, 16
dev = torch.device("cuda:0")
xs = [torch.randn(n, device=dev).to(torch.bfloat16) for _ in range(R)]
ys = [torch.empty_like(x) for x in xs]
cs = [torch.empty(n // 2, dtype=torch.uint8, device=dev) for _ in range(R)]
ss = [torch.empty(n // 128, dtype=torch.float32, device=dev) for _ in range(R)]
sp = torch.cuda.current_stream().cuda_stream
f = lambda i: L.lib.agq_quantize_roundtrip(xs[i].data_ptr(), 1, n, 4, 128, 0, cs[i].data_ptr(), 0, ss[i].data_ptr(), ys[i].data_ptr(), 1, None, sp)
for i in range(R): f(i)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for i in range(80): f(i % R)
e.record(); torch.cuda.synchronize()
print(round(s.elapsed_time(e) * 1e3 / 80, 2))
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for rnd in range(3):
    for lib in sys.argv[1:]:
        r = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, AGQ_LIB=lib, ROOT=root),
                           capture_output=True, text=True)
        print(rnd, lib.split("/")[-2], r.stdout.strip() or r.stderr[-300:], flush=True)
