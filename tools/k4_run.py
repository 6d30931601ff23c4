"""K4 alone for profiling: the P-piece local reduce-requant over a 2^27-element
chunk (tools/microbench.py's reduce case), 3 launches."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200 import _lib as L  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n = 1 << 27
dev = torch.device("cuda:0")
pieces = [A.quantize_blockwise(torch.randn(n, device=dev) * 1e-3, 8, 128, A.CodecKind.Fp8E4M3,
                               packed=False, check=False) for _ in range(P)]
oc, os_ = torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n // 128, device=dev)
err = A.ErrorRecord(dev).reset()
pc = L.ptr_array([p.codes.data_ptr() for p in pieces])
ps = L.ptr_array([p.scales.data_ptr() for p in pieces])
sp = torch.cuda.current_stream().cuda_stream
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
for i in range(3):
    if i == 2:
        s.record()
    L.check(L.lib.agq_fp8_reduce_requant(P, pc, ps, n, 128, 1, L.ptr_array([oc.data_ptr()]),
                                         L.ptr_array([os_.data_ptr()]), err.ptr, sp))
e.record()
torch.cuda.synchronize()
L.errors_message(err.read(), L.AGQ_OP_ALLREDUCE)
print(f"P={P} n={n} last launch {s.elapsed_time(e) * 1e3:.1f} us, "
      f"{n * (P + 1) * (1 + 4 / 128) / (s.elapsed_time(e) * 1e-3) / 1e9:.0f} GB/s")
