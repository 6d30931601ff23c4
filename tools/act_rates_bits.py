"""C2-silu-sized (235M BF16) quantize / dequantize at every width 4-8: us and GB/s."""
import json, os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2605_00539_b200 as A
from paper_2605_00539_b200 import _lib as L
dev = torch.device("cuda:0"); sp = torch.cuda.current_stream().cuda_stream
n = 16384 * 14336
x = torch.randn(n, device=dev).to(torch.bfloat16)
y = torch.empty_like(x)
for b in (4, 5, 6, 7, 8):
    c = torch.empty(n * b // 8, dtype=torch.uint8, device=dev); s = torch.empty(n // 128, device=dev)
    L.lib.agq_quantize(x.data_ptr(), 1, n, b, 128, 0, c.data_ptr(), 0, s.data_ptr(), None, sp)
    def q(): L.lib.agq_quantize(x.data_ptr(), 1, n, b, 128, 0, c.data_ptr(), 0, s.data_ptr(), None, sp)
    def d(): L.lib.agq_dequantize(c.data_ptr(), 0, s.data_ptr(), n, b, 128, 0, y.data_ptr(), 1, 0, None, sp)
    res = {}
    for name, f in (("q", q), ("d", d)):
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(10): f()
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 10 * 1e3
        byts = n * (2 + b / 8 + 4 / 128)
        res[name] = (round(us, 1), round(byts / us / 1e3, 1))
    print(b, res)
