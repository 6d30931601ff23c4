"""Per-kernel timing of the hot path on one B200 (CUDA events, warm, L2
flushed by rotating buffers larger than L2). Prints one line per case:
algorithmic GB/s and the fraction of the measured HBM copy peak."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2605_00539_b200 as A  # noqa: E402
from paper_2605_00539_b200 import _lib as L  # noqa: E402

PEAK = 6540.8


def timeit(fn, iters=20, warm=3):
    for _ in range(warm):
        fn(0)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for i in range(iters):
        fn(i)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="all")
    ap.add_argument("--n", type=int, default=0, help="act: single size")
    ap.add_argument("--bits", type=int, default=0, help="act: single width")
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    res = []
    stream = torch.cuda.current_stream().cuda_stream

    def report(name, sec, nbytes, extra=None):
        gbs = nbytes / sec / 1e9
        r = {"case": name, "us": round(sec * 1e6, 2), "GBs": round(gbs, 1), "frac": round(gbs / PEAK, 3)}
        if extra:
            r.update(extra)
        res.append(r)
        print(json.dumps(r), flush=True)

    if args.which in ("all", "act"):
        # C1: 4096^2 and C2-sized tensors, rotating copies to defeat L2
        sizes = ((4096 * 4096, "C1"), (16384 * 14336, "C2silu"))
        if args.n:
            sizes = ((args.n, f"n{args.n}"),)
        for n, label in sizes:
            R = max(2, int(1.2e9 // (n * 2)) + 1)
            xs = [torch.randn(n, device=dev).to(torch.bfloat16) for _ in range(R)]
            for bits in ((args.bits,) if args.bits else (4, 5, 6, 7, 8)):
                qs = [A.quantize_blockwise(x, bits, check=False) for x in xs]
                outs = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(R)]
                nq = n * 2 + n * bits / 8 + n / 128 * 4
                def fq(i):
                    x, q = xs[i % R], qs[i % R]
                    L.lib.agq_quantize(x.data_ptr(), L.AGQ_BF16, n, bits, 128, 0, q.codes.data_ptr(),
                                       L.AGQ_CODES_PACKED, q.scales.data_ptr(), None, stream)
                def fd(i):
                    q, o = qs[i % R], outs[i % R]
                    L.lib.agq_dequantize(q.codes.data_ptr(), L.AGQ_CODES_PACKED, q.scales.data_ptr(), n,
                                         bits, 128, 0, o.data_ptr(), L.AGQ_BF16, 0, None, stream)
                report(f"{label}_quant_b{bits}", timeit(fq, args.iters), nq)
                report(f"{label}_dequant_b{bits}", timeit(fd, args.iters), nq)
            del xs, qs, outs
            torch.cuda.empty_cache()
    if args.which in ("all", "acc"):
        n = 1 << 28
        R = 2
        mains = [A.quantize_blockwise(torch.randn(n, device=dev) * 1e-3, 8, 128, A.CodecKind.Fp8E4M3,
                                      packed=False, check=False) for _ in range(R)]
        locs = [torch.randn(n, device=dev) * 1e-3 for _ in range(R)]
        err = A.ErrorRecord(dev).reset()
        for prec in (0, 1, 2):
            def fa(i):
                m, l = mains[i % R], locs[i % R]
                L.lib.agq_fp8_accumulate(m.codes.data_ptr(), m.scales.data_ptr(), l.data_ptr(), L.AGQ_F32, n,
                                         128, prec, m.codes.data_ptr(), m.scales.data_ptr(), err.ptr, stream)
            report(f"acc_f32local_p{prec}", timeit(fa, 10), n * (1 + 4 + 1 + 8 / 128))
        lb = [l.to(torch.bfloat16) for l in locs]
        del locs
        def fb(i):
            m, l = mains[i % R], lb[i % R]
            L.lib.agq_fp8_accumulate(m.codes.data_ptr(), m.scales.data_ptr(), l.data_ptr(), L.AGQ_BF16, n,
                                     128, 0, m.codes.data_ptr(), m.scales.data_ptr(), err.ptr, stream)
        report("acc_bf16local", timeit(fb, 10), n * (1 + 2 + 1 + 8 / 128))
        h = err.read()
        print("errors:", h.nonfinite_block, h.bad_scale_block, h.nonfinite_local)
        del mains, lb
        torch.cuda.empty_cache()
    if args.which in ("all", "reduce"):
        n = 1 << 27
        for P in (2, 4, 8):
            pieces = [A.quantize_blockwise(torch.randn(n, device=dev) * 1e-3, 8, 128, A.CodecKind.Fp8E4M3,
                                           packed=False, check=False) for _ in range(P)]
            out = A.QuantizedTensor(torch.empty_like(pieces[0].codes), torch.empty_like(pieces[0].scales), 8)
            err = A.ErrorRecord(dev).reset()
            pc = L.ptr_array([p.codes.data_ptr() for p in pieces])
            ps = L.ptr_array([p.scales.data_ptr() for p in pieces])
            oc = L.ptr_array([out.codes.data_ptr()])
            os_ = L.ptr_array([out.scales.data_ptr()])
            def fr(i):
                L.lib.agq_fp8_reduce_requant(P, pc, ps, n, 128, 1, oc, os_, err.ptr, stream)
            report(f"reduce_P{P}", timeit(fr, 10), n * (P + 1) * (1 + 4 / 128))
            del pieces, out
            torch.cuda.empty_cache()
    print("launches", A.launch_count())


if __name__ == "__main__":
    main()
