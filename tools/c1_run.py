"""C1 round trips (INT4 quantize + dequantize of 16 rotating 4096^2 BF16
tensors) for profiling: prints the event-timed us per round trip."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_00539_b200 as A  # noqa: E402,F401
from paper_2605_00539_b200 import _lib as L  # noqa: E402

n, R = 4096 * 4096, 16
dev = torch.device("cuda:0")
xs = [torch.randn(n, device=dev).to(torch.bfloat16) for _ in range(R)]
ys = [torch.empty_like(x) for x in xs]
cs = [torch.empty(n // 2, dtype=torch.uint8, device=dev) for _ in range(R)]
ss = [torch.empty(n // 128, dtype=torch.float32, device=dev) for _ in range(R)]
sp = torch.cuda.current_stream().cuda_stream


def rt(i):
    L.check(L.lib.agq_quantize(xs[i].data_ptr(), L.AGQ_BF16, n, 4, 128, 0, cs[i].data_ptr(),
                               L.AGQ_CODES_PACKED, ss[i].data_ptr(), None, sp))
    L.check(L.lib.agq_dequantize(cs[i].data_ptr(), L.AGQ_CODES_PACKED, ss[i].data_ptr(), n, 4, 128,
                                 0, ys[i].data_ptr(), L.AGQ_BF16, 0, None, sp))


iters = int(sys.argv[1]) if len(sys.argv) > 1 else 80
for i in range(R):
    rt(i)
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for i in range(iters):
    rt(i % R)
e.record()
torch.cuda.synchronize()
print(f"C1 round trip {s.elapsed_time(e) * 1e3 / iters:.2f} us")
