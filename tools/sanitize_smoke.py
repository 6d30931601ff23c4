"""Small run of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck): act quant/dequant (all widths, bf16/f32, packed/bytes, tails,
generic block sizes, grouped), FP8 accumulate (f32/bf16 local, 3 precisions),
reduce-requant (P=1..8 and generic), naive ring, pack/unpack."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_00539_b200 as A  # noqa: E402

dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
for n in (8192 * 2 + 300, 1000):
    x = torch.randn(n, device=dev, generator=g)
    for dt in (torch.bfloat16, torch.float32):
        xx = x.to(dt)
        for kind, bits in [(A.CodecKind.SymmetricLinear, b) for b in (4, 5, 6, 7, 8)] + \
                          [(A.CodecKind.Fp4E2M1, 4), (A.CodecKind.Fp8E4M3, 8)]:
            for packed in (True, False):
                q = A.quantize_blockwise(xx, bits, 128, kind, packed=packed)
                A.dequantize_blockwise(q, torch.bfloat16)
                A.dequantize_blockwise(q, torch.float32)
            A.quantize_blockwise(xx, bits, 100, kind)
qs = A.quantize_grouped([torch.randn(n, device=dev, generator=g).to(torch.bfloat16)
                         for n in (8192 * 3, 5000)], 5)
A.dequantize_grouped(qs)
n = 8192 * 2 + 512
mains = [A.quantize_blockwise(torch.randn(n, device=dev, generator=g) * 1e-3, 8, 128,
                              A.CodecKind.Fp8E4M3, packed=False) for _ in range(8)]
for ldt in (torch.float32, torch.bfloat16):
    loc = (torch.randn(n, device=dev, generator=g) * 1e-3).to(ldt)
    for prec in range(3):
        A.local_accumulate(mains[0], loc, A.AccumulatePrecision(prec))
for P in range(1, 9):
    A.allreduce_simulated(mains[:P])
A.allreduce_naive_simulated(mains[:4])
c = torch.randint(0, 32, (5003,), device=dev, dtype=torch.uint8)
A.unpack_codes(A.pack_codes(c, 5), 5, 5003)
torch.cuda.synchronize()
print("sanitize smoke ok, launches", A.launch_count())
