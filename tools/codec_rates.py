"""Quantize / dequantize GB/s of every activation codec on a C2-sized BF16
tensor (235M elements, rotating copies > L2), CUDA events."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200 import _lib as L  # noqa: E402


def timeit(fn, iters=10):
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for i in range(iters):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) * 1e-3 / iters


F32 = "--f32" in sys.argv  # FP32 activations (the C++ drop-in surface's input type)
BYTES = "--bytes" in sys.argv  # one code per byte (the reference's host layout)
n = 16384 * 14336
dev = torch.device("cuda")
R = 3
xs = [torch.randn(n, device=dev).to(torch.float32 if F32 else torch.bfloat16) for _ in range(R)]
ESZ = 4 if F32 else 2
DT = L.AGQ_F32 if F32 else L.AGQ_BF16
sp = torch.cuda.current_stream().cuda_stream
for name, codec, bits in (("linear", 0, 4), ("linear", 0, 8), ("fp4_e2m1", 1, 4), ("fp8_e4m3", 2, 8)):
    qs = [A.quantize_blockwise(x, bits, 128, A.CodecKind(codec), packed=not BYTES, check=False)
          for x in xs]
    CL = L.AGQ_CODES_BYTES if BYTES else L.AGQ_CODES_PACKED
    outs = [torch.empty_like(xs[0]) for _ in range(R)]
    nb = n * ESZ + n * (1 if BYTES else bits / 8) + n / 128 * 4

    def fq(i):
        x, q = xs[i % R], qs[i % R]
        L.check(L.lib.agq_quantize(x.data_ptr(), DT, n, bits, 128, codec, q.codes.data_ptr(),
                                   CL, q.scales.data_ptr(), None, sp))

    def fd(i):
        q, o = qs[i % R], outs[i % R]
        L.check(L.lib.agq_dequantize(q.codes.data_ptr(), CL, q.scales.data_ptr(), n,
                                     bits, 128, codec, o.data_ptr(), DT, 0, None, sp))
    tq, td = timeit(fq), timeit(fd)
    print(json.dumps({"input": "f32" if F32 else "bf16", "codes": "bytes" if BYTES else "packed",
                      "codec": name, "bits": bits, "quant_GBs": round(nb / tq / 1e9, 1),
                      "dequant_GBs": round(nb / td / 1e9, 1)}), flush=True)
