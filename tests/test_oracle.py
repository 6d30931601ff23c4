"""Pin the CPU oracle (oracle/agq_oracle.c) before trusting it: against the
reference's own known-answer tests (proj/tests/test_*.cpp), against the
golden fixture produced by the reference itself (tests/golden/), and against
the reference compiled as-is (oracle/_ref) on random inputs."""
import math

import numpy as np
import pytest

import oracle_ffi as O

CODECS = [(O.LINEAR, b) for b in (4, 5, 6, 7, 8)] + [(O.FP4, 4), (O.FP8, 8)]


# ---- fp8 / fp4 scalars (test_fp8.cpp) -------------------------------------
def test_fp8_kats():
    enc = lambda v: O.orc.oracle_fp8_encode(v, None)
    assert enc(0.0) == 0x00 and enc(-0.0) == 0x80                      # :9-15
    ov = O.C.c_int(0)
    assert O.orc.oracle_fp8_encode(448.0, O.C.byref(ov)) == 0x7E and ov.value == 0
    assert O.orc.oracle_fp8_encode(500.0, O.C.byref(ov)) == 0x7E and ov.value == 1
    assert O.orc.oracle_fp8_encode(-500.0, O.C.byref(ov)) == 0xFE and ov.value == 1
    assert enc(432.0) == 0x7E                                           # :54-64
    assert O.orc.oracle_fp8_decode(enc(431.0)) == 416.0
    assert O.orc.oracle_fp8_decode(enc(433.0)) == 448.0
    assert O.orc.oracle_fp8_decode(enc(21.0)) == 20.0
    assert enc(2.0 ** -10) == 0x00
    assert O.orc.oracle_fp8_decode(enc(0.002)) == 2.0 ** -9


def test_fp8_exhaustive_roundtrip_and_monotone():
    for b in range(256):                                                # :34-43
        x = O.orc.oracle_fp8_decode(b)
        assert O.orc.oracle_fp8_encode(x, None) == b
    vals = [O.orc.oracle_fp8_decode(b) for b in range(0x7F)]
    assert all(b > a for a, b in zip(vals, vals[1:]))                   # :45-52


def test_fp8_dense_grid_nearest():
    grid = np.array([O.orc.oracle_fp8_decode(b) for b in range(0x7F)])
    for x in np.arange(0.0, 448.0, 0.37):                               # :66-77
        got = O.orc.oracle_fp8_decode(O.orc.oracle_fp8_encode(float(x), None))
        assert abs(abs(x - got) - np.min(np.abs(x - grid))) < 1e-12


def test_fp4_kats():
    grid = [0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0]                      # test_fp8.cpp:85-97
    for i, g in enumerate(grid):
        assert O.orc.oracle_fp4_decode(O.orc.oracle_fp4_encode(g)) == g
        if i:
            assert O.orc.oracle_fp4_decode(O.orc.oracle_fp4_encode(-g)) == -g
    d = lambda v: O.orc.oracle_fp4_decode(O.orc.oracle_fp4_encode(v))
    assert (d(0.25), d(0.75), d(2.5), d(5.0), d(100.0)) == (0.0, 1.0, 2.0, 4.0, 6.0)
    assert O.orc.oracle_fp4_encode(-0.0) == 0


def test_scalars_match_golden(golden):
    assert np.array_equal(np.array([O.orc.oracle_fp8_decode(b) for b in range(256)]),
                          golden["fp8_decode"], equal_nan=True)
    assert [O.orc.oracle_fp8_encode(float(v), None) for v in golden["fp8_probe"]] == \
        list(golden["fp8_probe_codes"])
    assert [O.orc.oracle_fp4_encode(float(v)) for v in golden["fp4_probe"]] == \
        list(golden["fp4_probe_codes"])
    rin = golden["round_in"]
    assert np.array_equal(np.array([O.orc.oracle_round_bf16(v) for v in rin], np.float32),
                          golden["round_bf16"])
    assert np.array_equal(np.array([O.orc.oracle_round_fp16(v) for v in rin], np.float32),
                          golden["round_fp16"])


# ---- block codec ---------------------------------------------------------
@pytest.mark.parametrize("name", ["x_cli", "x_cli_bf16", "x_codec", "x_ragged"])
def test_codec_matches_golden(golden, name):
    x = golden[name]
    for codec, bits in CODECS:
        for block in (128, 16, 1000):
            key = f"{name}_c{codec}_b{bits}_k{block}"
            c, s = O.quantize(x, bits, block, codec)
            assert np.array_equal(c, golden[key + "_codes"]), key
            assert np.array_equal(s, golden[key + "_scales"]), key
            d = O.dequantize(c, s, bits, block, codec)
            assert np.array_equal(d.view(np.uint32), golden[key + "_deq"].view(np.uint32)), key
            assert np.array_equal(O.pack(c, bits), golden[key + "_packed"]), key
            assert np.array_equal(O.unpack(golden[key + "_packed"], bits, x.size), c)


@pytest.mark.skipif(O.ref is None, reason="reference not built here")
def test_codec_matches_reference_random():
    rng = np.random.default_rng(5)
    for trial in range(12):
        n = int(rng.integers(1, 5000))
        x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-8, 8)).astype(np.float32)
        if trial % 3 == 0:
            x = O.bf16_round(x)
        if trial % 4 == 1:
            x[rng.integers(0, n, size=n // 7)] = 0.0
        block = int(rng.choice([1, 2, 16, 128, 129, 1000]))
        for codec, bits in CODECS:
            c0, s0 = O.quantize(x, bits, block, codec, lib=O.ref)
            c1, s1 = O.quantize(x, bits, block, codec)
            assert np.array_equal(c0, c1) and np.array_equal(s0, s1)
            d0 = O.dequantize(c0, s0, bits, block, codec, lib=O.ref)
            d1 = O.dequantize(c0, s0, bits, block, codec)
            assert np.array_equal(d0.view(np.uint32), d1.view(np.uint32))


def test_codec_error_texts():
    x = np.ones(16, np.float32)
    for bits, block, codec in ((3, 128, 0), (9, 128, 0), (4, 0, 0), (5, 128, 2), (5, 128, 1)):
        with pytest.raises(O.OracleError) as e:                         # test_codec.cpp:199-208
            O.quantize(x, bits, block, codec)
        assert e.value.status == 1
    y = np.random.default_rng(8).standard_normal(300).astype(np.float32)
    y[170] = np.inf
    with pytest.raises(O.OracleError, match="block 1"):                 # :162-171
        O.quantize(y, 4, 128)


def test_codec_properties():
    x = np.zeros(300, np.float32)                                       # :26-40
    for codec, bits in ((0, 5), (1, 4), (2, 8)):
        c, s = O.quantize(x, bits, 128, codec)
        assert np.all(s == 0)
        assert np.all(O.dequantize(c, s, bits, 128, codec) == 0)
    x = np.zeros(130, np.float32)                                       # :173-184
    x[:128] = 8.0
    x[128], x[129] = 0.5, -1.0
    c, s = O.quantize(x, 4, 128)
    assert list(s) == [8.0, 1.0]
    assert O.dequantize(c, s, 4)[129] == -1.0
    rng = np.random.default_rng(1)
    x = rng.standard_normal(4096).astype(np.float32)
    for bits in range(4, 9):                                            # :61-75
        c, s = O.quantize(x, bits, 128)
        d = O.dequantize(c, s, bits)
        L = (1 << (bits - 1)) - 1
        sc = np.repeat(s, 128)[: x.size].astype(np.float64)
        assert np.all(np.abs(d.astype(np.float64) - x) <= sc / (2 * L) + sc * 1.2e-7)


def test_dump_golden(golden):
    x = np.array([1.0, -1.0, 0.5], np.float32)
    c, s = O.quantize(x, 4, 2)
    out = np.zeros(O.orc.oracle_dump_size(3, 4, 2, 1), np.uint8)
    shape = np.array([3], np.uint64)
    k = O.orc.oracle_dump(O._p(c), O._p(s), 3, 4, 2, 0, O._p(shape), 1, O._p(out))
    assert np.array_equal(out[:k], golden["dump_3_b4_k2"])
    assert bytes(out[:4]) == b"AGQT" and out[-2] == 14 and out[-1] == 14  # test_codec.cpp:244-264
    x = golden["x777"]
    c, s = O.quantize(x, 6, 128)
    out = np.zeros(O.orc.oracle_dump_size(777, 6, 128, 2), np.uint8)
    shape = np.array([7, 111], np.uint64)
    k = O.orc.oracle_dump(O._p(c), O._p(s), 777, 6, 128, 0, O._p(shape), 2, O._p(out))
    assert np.array_equal(out[:k], golden["dump_777_b6"])


# ---- gradient path -------------------------------------------------------
def test_local_accumulate_golden(golden):
    for prec in (0, 1, 2):
        oc, os_ = O.local_accumulate(golden["acc_main_codes"], golden["acc_main_scales"],
                                     golden["acc_local"], prec)
        assert np.array_equal(oc, golden[f"acc_p{prec}_codes"])
        assert np.array_equal(os_, golden[f"acc_p{prec}_scales"])


def test_local_accumulate_kats():
    z = np.zeros(256, np.float32)                                       # test_collective.cpp:50-62
    g = np.random.default_rng(2).standard_normal(256).astype(np.float32)
    mc, ms = O.quantize(z, 8, 128, O.FP8)
    oc, os_ = O.local_accumulate(mc, ms, g)
    dc, ds = O.quantize(g, 8, 128, O.FP8)
    assert np.array_equal(oc, dc) and np.array_equal(os_, ds)
    c, s = O.quantize(np.zeros(128, np.float32), 8, 128, O.FP8)          # :64-82
    for _ in range(8):
        c, s = O.local_accumulate(c, s, np.full(128, 100.0, np.float32))
    assert np.all(O.dequantize(c, s, 8, 128, O.FP8) == 800.0)
    c, s = O.quantize(np.full(128, 2.0, np.float32), 8, 128, O.FP8)       # :122-135
    for prec in (1, 2):
        oc, os_ = O.local_accumulate(c, s, np.ones(128, np.float32), prec)
        assert O.dequantize(oc, os_, 8, 128, O.FP8)[0] == 3.0
    bad = np.zeros(128, np.float32)
    bad[5] = np.nan
    with pytest.raises(O.OracleError, match="non-finite local gradient element"):
        O.local_accumulate(c, s, bad)


def test_round_fp16_kats():
    assert O.orc.oracle_round_bf16(1.0039062) == 1.0
    assert O.orc.oracle_round_fp16(65504.0) == 65504.0
    assert O.orc.oracle_round_fp16(70000.0) == 65504.0


def test_chunk_assignment_kats():
    r = np.zeros(8, np.uint64)
    O.orc.oracle_chunk_assignment(4096, 128, 4, O._p(r))                # test_collective.cpp:38-48
    assert list(r[:2]) == [0, 1024] and list(r[6:8]) == [3072, 4096]
    O.orc.oracle_chunk_assignment(300, 128, 2, O._p(r))
    assert list(r[:4]) == [0, 256, 256, 300]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_allreduce_golden(golden, world):
    codes = list(golden[f"ar{world}_in_codes"])
    scales = list(golden[f"ar{world}_in_scales"])
    oc, os_ = O.allreduce_decomposed(codes, scales)
    assert np.array_equal(oc, golden[f"ar{world}_codes"])
    assert np.array_equal(os_, golden[f"ar{world}_scales"])
    # == quantize(allreduce_oracle) bit-exactly (test_collective.cpp:203-216)
    acc = O.allreduce_oracle(codes, scales)
    dc, ds = O.quantize(acc, 8, 128, O.FP8)
    assert np.array_equal(oc, dc) and np.array_equal(os_, ds)
    nc, ns, ov = O.allreduce_naive(codes, scales)
    assert np.array_equal(nc, golden[f"naive{world}_codes"])
    assert np.array_equal(ns, golden[f"naive{world}_scales"])
    assert ov == int(golden[f"naive{world}_overflow"][0])


def test_allreduce_constant64_and_signed_zero(golden):
    c, s = O.quantize(np.full(512, 64.0, np.float32), 8, 128, O.FP8)
    oc, os_ = O.allreduce_decomposed([c] * 8, [s] * 8)
    assert np.all(O.dequantize(oc, os_, 8, 128, O.FP8) == 512.0)
    nc, ns, ov = O.allreduce_naive([c] * 8, [s] * 8)
    assert ov == 512 and np.all(O.dequantize(nc, ns, 8, 128, O.FP8) == 64.0)
    assert np.array_equal(nc, golden["c64_naive_codes"])
    assert golden["sz_in_codes"][5] == 0x80
    for P in (1, 2):
        oc, os_ = O.allreduce_decomposed([golden["sz_in_codes"]] * P, [golden["sz_in_scales"]] * P)
        assert np.array_equal(oc, golden[f"sz{P}_codes"])
        assert oc[5] == 0x00


@pytest.mark.skipif(O.ref is None, reason="reference not built here")
def test_allreduce_matches_reference_random():
    rng = np.random.default_rng(3)
    for world in (1, 2, 3, 5, 8):
        n = int(rng.integers(1, 3000))
        codes, scales = [], []
        for r in range(world):
            c, s = O.quantize((rng.standard_normal(n) * 1e-2).astype(np.float32), 8, 128, O.FP8)
            codes.append(c)
            scales.append(s)
        r0 = O.ref_allreduce(0, codes, scales)
        oc, os_ = O.allreduce_decomposed(codes, scales)
        assert np.array_equal(oc, r0[0]) and np.array_equal(os_, r0[1])
        r1 = O.ref_allreduce(1, codes, scales)
        nc, ns, ov = O.allreduce_naive(codes, scales)
        assert np.array_equal(nc, r1[0]) and np.array_equal(ns, r1[1]) and ov == r1[2]


# ---- DBCA planner (test_dbca.cpp) ------------------------------------------
def _plan(n, mb):
    c = (O.C.c_int * n)()
    r = (O.C.c_double * n)()
    a = (O.C.c_int * n)()
    st = O.orc.oracle_plan_bit_widths(n, mb, 2, c, r, a)
    return st, list(c), list(r), list(a)


def test_dbca_kats():
    assert _plan(4, 8)[1] == [11, 9, 7, 5]
    assert _plan(8, 16)[1] == [23, 21, 19, 17, 15, 13, 11, 9]
    assert _plan(1, 1)[1] == [1]
    assert _plan(4, 6)[0] != 0
    st, c, r, a = _plan(4, 8)
    assert a == [4, 5, 6, 8] and math.isclose(r[1], 44 / 9) and math.isclose(r[3], 8.8)
    assert _plan(2, 4)[1] == [5, 3] and _plan(2, 4)[3] == [4, 7]
    assert _plan(8, 16)[3] == [4, 4, 5, 5, 6, 7, 8, 8]
    ap = (O.C.c_int * 8)()
    pk, u4, ok = O.C.c_double(), O.C.c_double(), O.C.c_int()
    O.orc.oracle_plan_reuse(4, 8, 8, 16, ap, O.C.byref(pk), O.C.byref(u4), O.C.byref(ok))
    assert list(ap) == [4, 4, 4, 4, 4, 5, 6, 8] and u4.value == 92.0 and ok.value == 1
