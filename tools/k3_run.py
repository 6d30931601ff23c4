"""K3 alone for profiling: FP8 local_accumulate over 2^28 elements with a
BF16 (argv[1] = bf16) or FP32 local gradient and precision argv[2]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200 import _lib as L  # noqa: E402

ldt = sys.argv[1] if len(sys.argv) > 1 else "bf16"
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = 1 << 28
dev = torch.device("cuda:0")
m = A.quantize_blockwise(torch.randn(n, device=dev) * 1e-3, 8, 128, A.CodecKind.Fp8E4M3,
                         packed=False, check=False)
loc = (torch.randn(n, device=dev) * 1e-3).to(torch.bfloat16 if ldt == "bf16" else torch.float32)
err = A.ErrorRecord(dev).reset()
sp = torch.cuda.current_stream().cuda_stream
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
for i in range(3):
    if i == 2:
        s.record()
    L.check(L.lib.agq_fp8_accumulate(m.codes.data_ptr(), m.scales.data_ptr(), loc.data_ptr(),
                                     L.AGQ_BF16 if ldt == "bf16" else L.AGQ_F32, n, 128, prec,
                                     m.codes.data_ptr(), m.scales.data_ptr(), err.ptr, sp))
e.record()
torch.cuda.synchronize()
L.errors_message(err.read(), L.AGQ_OP_ACCUMULATE)
print(f"K3 {ldt} prec={prec} n={n}: {s.elapsed_time(e) * 1e3:.1f} us")
