"""Generate tests/golden/golden.npz from the REFERENCE ITSELF.

Runs only where oracle/_ref/libagq_ref.so exists (built from the unmodified
reference headers by oracle/Makefile). Every array in the fixture is an output
of the reference's own functions on inputs drawn with the reference's RNG
(agq::make_rng + std::normal_distribution<float>, libstdc++ of this image):

  python tests/golden/make_golden.py

The fixture pins the C oracle (tests/test_oracle.py) and the GPU kernels
(tests/test_gpu_*.py) on machines where /root/reference is absent.
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle_ffi as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main():
    if O.ref is None:
        raise SystemExit("oracle/_ref/libagq_ref.so missing: run `make -C oracle` here")
    R = O.ref
    g = {}
    # ---- inputs: agq CLI `quantize --normal 4096` (agq.cpp:47-65, seed 1)
    x = O.ref_normal(1, 0x1D, 0, 4096)
    xb = O.bf16_round(x)
    g["x_cli"] = x
    g["x_cli_bf16"] = xb
    # test_codec.cpp:15-22 random_floats(4096, 1234)
    g["x_codec"] = O.ref_normal_seed(1234, 4096)
    # ragged + special values
    xr = O.ref_normal(7, 0x1D, 0, 1000) * np.float32(3.0)
    xr[:128] = 0.0
    xr[200] = np.float32(-0.0)
    xr[300] = np.float32(1e-30)
    g["x_ragged"] = xr
    for name in ("x_cli", "x_cli_bf16", "x_codec", "x_ragged"):
        src = g[name]
        for codec, bits_list in ((O.LINEAR, (4, 5, 6, 7, 8)), (O.FP4, (4,)), (O.FP8, (8,))):
            for bits in bits_list:
                for block in (128, 16, 1000):
                    c, s = O.quantize(src, bits, block, codec, lib=R)
                    key = f"{name}_c{codec}_b{bits}_k{block}"
                    g[key + "_codes"] = c
                    g[key + "_scales"] = s
                    g[key + "_deq"] = O.dequantize(c, s, bits, block, codec, lib=R)
                    g[key + "_packed"] = O.pack(c, bits, lib=R)
    # ---- AGQT dump header golden (test_codec.cpp:244-264)
    x3 = np.array([1.0, -1.0, 0.5], np.float32)
    buf = np.zeros(256, np.uint8)
    shape = np.array([3], np.uint64)
    k = R.ref_dump_quantized(O._p(x3), 3, 4, 2, 0, O._p(shape), 1, O._p(buf), 256)
    g["dump_3_b4_k2"] = buf[:k].copy()
    x777 = O.ref_normal_seed(55, 777)
    shape = np.array([7, 111], np.uint64)
    big = np.zeros(16384, np.uint8)
    k = R.ref_dump_quantized(O._p(x777), 777, 6, 128, 0, O._p(shape), 2, O._p(big), 16384)
    g["dump_777_b6"] = big[:k].copy()
    g["x777"] = x777
    # ---- scalar formats
    g["fp8_decode"] = np.array([R.ref_fp8_decode(b) for b in range(256)])
    probe = [0.0, -0.0, 448.0, 500.0, -500.0, 432.0, 431.0, 433.0, 21.0, 2.0 ** -10, 0.002]
    g["fp8_probe"] = np.array(probe)
    g["fp8_probe_codes"] = np.array([R.ref_fp8_encode(v, None) for v in probe], np.uint8)
    g["fp4_probe"] = np.array([0.25, 0.75, 2.5, 5.0, 100.0, -0.0, -1.25, 3.4])
    g["fp4_probe_codes"] = np.array([R.ref_fp4_encode(v) for v in g["fp4_probe"]], np.uint8)
    rb = np.array([1.0, 1.0039062, 65504.0, 70000.0, 0.0, -3.14159, 1e-7, 6.1e-5], np.float32)
    g["round_in"] = rb
    g["round_bf16"] = np.array([R.ref_round_bf16(v) for v in rb], np.float32)
    g["round_fp16"] = np.array([R.ref_round_fp16(v) for v in rb], np.float32)
    # ---- local_accumulate (collective.hpp:128-147)
    n = 4096
    mainv = O.ref_normal(11, 3, 0, n, std=1e-3)
    mc, ms = O.quantize(mainv, 8, 128, O.FP8, lib=R)
    loc = O.ref_normal(11, 3, 1, n, std=1e-3)
    g["acc_main_codes"], g["acc_main_scales"], g["acc_local"] = mc, ms, loc
    for prec in (0, 1, 2):
        oc, os_ = O.local_accumulate(mc, ms, loc, prec, lib=R)
        g[f"acc_p{prec}_codes"], g[f"acc_p{prec}_scales"] = oc, os_
    # ---- decomposed all-reduce (test_collective.cpp:203-216 shapes)
    for world in (2, 4, 8):
        codes, scales = [], []
        for r in range(world):
            v = O.ref_normal(900 + world, 0xC0, r, 1024)
            c, s = O.quantize(v, 8, 128, O.FP8, lib=R)
            codes.append(c)
            scales.append(s)
        oc, os_, _, ev, same = O.ref_allreduce(0, codes, scales)
        assert same
        g[f"ar{world}_in_codes"] = np.stack(codes)
        g[f"ar{world}_in_scales"] = np.stack(scales)
        g[f"ar{world}_codes"], g[f"ar{world}_scales"] = oc, os_
        g[f"ar{world}_trace"] = ev
        oc, os_, ov, _, _ = O.ref_allreduce(1, codes, scales)
        g[f"naive{world}_codes"], g[f"naive{world}_scales"] = oc, os_
        g[f"naive{world}_overflow"] = np.array([ov], np.uint64)
    # ---- constant-64 separation (test_collective.cpp:160-181)
    c, s = O.quantize(np.full(512, 64.0, np.float32), 8, 128, O.FP8, lib=R)
    oc, os_, _, _, _ = O.ref_allreduce(0, [c] * 8, [s] * 8)
    g["c64_dec_codes"], g["c64_dec_scales"] = oc, os_
    oc, os_, ov, _, _ = O.ref_allreduce(1, [c] * 8, [s] * 8)
    g["c64_naive_codes"], g["c64_naive_scales"] = oc, os_
    g["c64_naive_overflow"] = np.array([ov], np.uint64)
    # ---- signed zero: x = -1e-9 at absmax 0.5 -> 0x80 in, 0x00 out
    xz = np.zeros(128, np.float32)
    xz[0] = 0.5
    xz[5] = -1e-9
    c, s = O.quantize(xz, 8, 128, O.FP8, lib=R)
    g["sz_in_codes"], g["sz_in_scales"] = c, s
    oc, os_, _, _, _ = O.ref_allreduce(0, [c, c], [s, s])
    g["sz2_codes"], g["sz2_scales"] = oc, os_
    oc, os_, _, _, _ = O.ref_allreduce(0, [c], [s])
    g["sz1_codes"], g["sz1_scales"] = oc, os_
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays, {os.path.getsize(OUT)} bytes")


if __name__ == "__main__":
    main()
