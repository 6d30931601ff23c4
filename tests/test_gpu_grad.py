"""GPU parity of the gradient path: fused FP8 local_accumulate (K3), the
decomposed all-reduce's reduce-requant (K4) in its one-device simulation,
and the naive FP8 ring — bit-exact against the reference golden fixture and
the C oracle, plus the reference's own property tests
(proj/tests/test_collective.cpp)."""
import numpy as np
import pytest
import torch

import oracle_ffi as O
import paper_2605_00539_b200 as A

pytestmark = pytest.mark.gpu
FP8 = A.CodecKind.Fp8E4M3


def t(x, dev, dtype=None):
    a = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    return a.to(dtype) if dtype is not None else a


def u32(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def fp8q(codes, scales, dev):
    return A.QuantizedTensor(t(codes, dev), t(scales, dev), 8, 128, (codes.size,), FP8, packed=False)


def same(q, codes, scales):
    assert np.array_equal(q.codes.cpu().numpy(), codes)
    assert np.array_equal(u32(q.scales.cpu().numpy()), u32(scales))


@pytest.mark.parametrize("prec", [0, 1, 2])
def test_accumulate_golden(cuda, golden, prec):
    main = fp8q(golden["acc_main_codes"], golden["acc_main_scales"], cuda)
    out = A.local_accumulate(main, t(golden["acc_local"], cuda), A.AccumulatePrecision(prec))
    same(out, golden[f"acc_p{prec}_codes"], golden[f"acc_p{prec}_scales"])


@pytest.mark.parametrize("n", [128, 8192, 8192 * 7 + 300, 200003])
@pytest.mark.parametrize("prec", [0, 1, 2])
@pytest.mark.parametrize("bf16_local", [False, True])
def test_accumulate_random(cuda, n, prec, bf16_local):
    rng = np.random.default_rng(n * 3 + prec)
    nb = (n + 127) // 128
    mag = np.repeat(10.0 ** rng.uniform(-8, 3, nb), 128)[:n]
    mag[:256] = 0.0  # zero main blocks
    mc, ms = O.quantize((rng.standard_normal(n) * mag).astype(np.float32), 8, 128, O.FP8)
    loc = (rng.standard_normal(n) * np.repeat(10.0 ** rng.uniform(-8, 3, nb), 128)[:n]).astype(np.float32)
    loc[:128] = 0.0  # 0 + 0 block
    loc[300:310] = -loc[300:310]
    if prec == 2:
        loc[1000:1010] = 7e4  # fp16 saturation path
    if bf16_local:
        loc = O.bf16_round(loc)
    oc, os_ = O.local_accumulate(mc, ms, loc, prec)
    lt = t(loc, cuda, torch.bfloat16 if bf16_local else torch.float32)
    for in_place in (False, True):
        main = fp8q(mc, ms, cuda)
        out = A.local_accumulate(main, lt, A.AccumulatePrecision(prec), in_place=in_place)
        same(out, oc, os_)


def test_accumulate_reference_properties(cuda):
    z = np.zeros(256, np.float32)                                   # test_collective.cpp:50-62
    g = np.random.default_rng(2).standard_normal(256).astype(np.float32)
    mc, ms = O.quantize(z, 8, 128, O.FP8)
    dc, ds = O.quantize(g, 8, 128, O.FP8)
    same(A.local_accumulate(fp8q(mc, ms, cuda), t(g, cuda)), dc, ds)
    mc, ms = O.quantize(np.zeros(128, np.float32), 8, 128, O.FP8)   # :64-82
    main = fp8q(mc, ms, cuda)
    c100 = t(np.full(128, 100.0, np.float32), cuda)
    for _ in range(8):
        main = A.local_accumulate(main, c100)
    assert torch.all(A.dequantize_blockwise(main) == 800.0)
    rel = []                                                        # :84-108
    for trial in range(5):
        rng = np.random.default_rng(500 + trial)
        main = fp8q(*O.quantize(np.zeros(1024, np.float32), 8, 128, O.FP8), cuda)
        oracle = np.zeros(1024, np.float32)
        for s in range(16):
            gs = rng.standard_normal(1024).astype(np.float32)
            main = A.local_accumulate(main, t(gs, cuda))
            oracle += gs
        v = A.dequantize_blockwise(main).cpu().numpy()
        rel.append(np.linalg.norm(v - oracle) / np.linalg.norm(oracle))
    assert max(rel) < 0.15


def test_accumulate_errors(cuda):
    mc, ms = O.quantize(np.ones(128, np.float32), 8, 128, O.FP8)
    g = np.zeros(128, np.float32)
    g[5] = np.nan
    with pytest.raises(A.InvalidArgument, match="non-finite local gradient element"):
        A.local_accumulate(fp8q(mc, ms, cuda), t(g, cuda))
    with pytest.raises(A.InvalidArgument, match="shape mismatch"):
        A.local_accumulate(fp8q(mc, ms, cuda), t(np.zeros(64, np.float32), cuda))
    lin = A.quantize_blockwise(t(np.zeros(128, np.float32), cuda), 8, 128, packed=False)
    with pytest.raises(A.InvalidArgument, match="FP8 E4M3"):
        A.local_accumulate(lin, t(np.zeros(128, np.float32), cuda))
    # fp32 overflow of the sum -> non-finite input in block k (quantize throws)
    big = np.full(8192 * 2, 3e38, np.float32)
    bc, bs = O.quantize(big, 8, 128, O.FP8)
    with pytest.raises(A.InvalidArgument, match="non-finite input element in block 0"):
        A.local_accumulate(fp8q(bc, bs, cuda), t(big, cuda))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_allreduce_golden(cuda, golden, world):
    mains = [fp8q(c, s, cuda) for c, s in zip(golden[f"ar{world}_in_codes"],
                                              golden[f"ar{world}_in_scales"])]
    same(A.allreduce_simulated(mains), golden[f"ar{world}_codes"], golden[f"ar{world}_scales"])
    out, ov = A.allreduce_naive_simulated(mains)
    same(out, golden[f"naive{world}_codes"], golden[f"naive{world}_scales"])
    assert ov == int(golden[f"naive{world}_overflow"][0])


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8, 11, 16])
def test_allreduce_random(cuda, world):
    rng = np.random.default_rng(world)
    n = 8192 * 3 + 200
    codes, scales = [], []
    for r in range(world):
        mag = np.repeat(10.0 ** rng.uniform(-6, 2, (n + 127) // 128), 128)[:n]
        c, s = O.quantize((rng.standard_normal(n) * mag).astype(np.float32), 8, 128, O.FP8)
        codes.append(c)
        scales.append(s)
    oc, os_ = O.allreduce_decomposed(codes, scales)
    same(A.allreduce_simulated([fp8q(c, s, cuda) for c, s in zip(codes, scales)]), oc, os_)
    if world <= 8:
        nc, ns, ov = O.allreduce_naive(codes, scales)
        out, gov = A.allreduce_naive_simulated([fp8q(c, s, cuda) for c, s in zip(codes, scales)])
        same(out, nc, ns)
        assert gov == ov


def test_allreduce_constant64_and_signed_zero(cuda, golden):
    c, s = O.quantize(np.full(512, 64.0, np.float32), 8, 128, O.FP8)
    mains = [fp8q(c, s, cuda)] * 8
    out = A.allreduce_simulated(mains)
    assert torch.all(A.dequantize_blockwise(out) == 512.0)             # exact 512
    nout, ov = A.allreduce_naive_simulated(mains)
    assert ov == 512 and torch.all(A.dequantize_blockwise(nout) == 64.0)
    for P in (1, 2):
        m = [fp8q(golden["sz_in_codes"], golden["sz_in_scales"], cuda)] * P
        o = A.allreduce_simulated(m)
        same(o, golden[f"sz{P}_codes"], golden[f"sz{P}_scales"])
        assert int(o.codes[5]) == 0x00


def test_allreduce_overflow_aborts(cuda):
    c, s = O.quantize(np.full(256, 3e38, np.float32), 8, 128, O.FP8)
    with pytest.raises(A.ProtocolError, match="fp32 overflow during local reduce"):
        A.allreduce_simulated([fp8q(c, s, cuda)] * 2)


def test_reduce_generic_block_sizes(cuda):
    rng = np.random.default_rng(7)
    for block in (2, 16, 100, 1000):
        n = 3001
        codes, scales = [], []
        for r in range(3):
            cc, ss = O.quantize(rng.standard_normal(n).astype(np.float32), 8, block, O.FP8)
            codes.append(cc)
            scales.append(ss)
        oc, os_ = O.allreduce_decomposed(codes, scales, block)
        mains = [A.QuantizedTensor(t(cc, cuda), t(ss, cuda), 8, block, (n,), FP8, packed=False)
                 for cc, ss in zip(codes, scales)]
        same(A.allreduce_simulated(mains), oc, os_)
        # generic accumulate with the same block
        loc = rng.standard_normal(n).astype(np.float32)
        ac, as_ = O.local_accumulate(codes[0], scales[0], loc, 0, block)
        same(A.local_accumulate(mains[0], t(loc, cuda)), ac, as_)


def test_second_allreduce_scales_by_world(cuda):
    rng = np.random.default_rng(55)                                 # test_collective.cpp:268-283
    codes, scales = zip(*[O.quantize(rng.standard_normal(512).astype(np.float32), 8, 128, O.FP8)
                          for _ in range(4)])
    first = A.allreduce_simulated([fp8q(c, s, cuda) for c, s in zip(codes, scales)])
    v1 = A.dequantize_blockwise(first).cpu().numpy()
    second = A.allreduce_simulated([first] * 4)
    v2 = A.dequantize_blockwise(second).cpu().numpy()
    step = np.repeat(second.scales.cpu().numpy(), 128) * (32.0 / 448.0)
    assert np.all(np.abs(v2 - 4.0 * v1) <= 4 * step + 1e-5)


def test_accumulate_beyond_2g_elements_sampled(cuda):
    """Config C3 class at > 2^31 elements (64-bit indexing): the whole buffer
    is processed on the GPU, blocks sampled around the 2^31 boundary and at
    random are checked bit-exact against the oracle."""
    n = (1 << 31) + 8192 * 3 + 256
    g = torch.Generator(device=cuda).manual_seed(3)
    x = torch.randn(n, device=cuda, generator=g) * 1e-3
    main = A.quantize_blockwise(x, 8, 128, FP8, packed=False)
    del x
    loc = torch.randn(n, device=cuda, generator=g) * 1e-3
    ref_codes = main.codes.clone()
    ref_scales = main.scales.clone()
    out = A.local_accumulate(main, loc, in_place=True)
    rng = np.random.default_rng(0)
    blocks = list(rng.integers(0, n // 128, 40)) + [(1 << 31) // 128 - 1, (1 << 31) // 128,
                                                    (1 << 31) // 128 + 1, n // 128]
    for b in blocks:
        lo, hi = b * 128, min(n, b * 128 + 128)
        oc, os_ = O.local_accumulate(ref_codes[lo:hi].cpu().numpy(), ref_scales[b:b + 1].cpu().numpy(),
                                     loc[lo:hi].cpu().numpy())
        assert np.array_equal(out.codes[lo:hi].cpu().numpy(), oc), b
        assert np.array_equal(u32(out.scales[b:b + 1].cpu().numpy()), u32(os_)), b


def test_allreduce_beyond_2g_elements_sampled(cuda):
    n = (1 << 31) + 1000
    g = torch.Generator(device=cuda).manual_seed(4)
    mains = []
    for _ in range(2):
        x = torch.randn(n, device=cuda, generator=g) * 1e-2
        mains.append(A.quantize_blockwise(x, 8, 128, FP8, packed=False))
        del x
    out = A.allreduce_simulated(mains)
    rng = np.random.default_rng(1)
    for b in list(rng.integers(0, n // 128, 30)) + [(1 << 31) // 128, n // 128]:
        lo, hi = b * 128, min(n, b * 128 + 128)
        oc, os_ = O.allreduce_decomposed([m.codes[lo:hi].cpu().numpy() for m in mains],
                                         [m.scales[b:b + 1].cpu().numpy() for m in mains])
        assert np.array_equal(out.codes[lo:hi].cpu().numpy(), oc), b
        assert np.array_equal(u32(out.scales[b:b + 1].cpu().numpy()), u32(os_)), b


def test_accumulate_encoder_exhaustive_bf16_domain(cuda):
    """K3's requantizer (hardware E4M3 conversion bracketed by +-2^-21, exact
    fallback) over every BF16 x <= a for every BF16 mantissa a: accumulate
    onto an all-zero FP8 main gradient (+0.0 + -0.0 = +0.0, so compare with
    the oracle's local_accumulate, not a direct quantize)."""
    mags = (np.arange(0x8000, dtype=np.uint32) << 16).view(np.float32)
    rows = []
    for am in range(128):
        a = np.array([(0x3F80 | am) << 16], np.uint32).view(np.float32)[0]
        xs = mags[mags <= a]
        xs = np.concatenate([xs, -xs])
        xs = np.concatenate([xs, np.zeros((-len(xs)) % 127, np.float32)]).reshape(-1, 127)
        rows.append(np.concatenate([np.full((xs.shape[0], 1), a, np.float32), xs], 1).reshape(-1))
    x = np.concatenate(rows)
    x = np.concatenate([x, np.zeros((-x.size) % 512, np.float32)])
    zc, zs = O.quantize(np.zeros(x.size, np.float32), 8, 128, O.FP8)
    out = A.local_accumulate(fp8q(zc, zs, cuda), t(x, cuda))
    c, s = O.local_accumulate(zc, zs, x)
    bad = np.nonzero(out.codes.cpu().numpy() != c)[0]
    assert bad.size == 0, (bad[:5], x[bad[:5]])
    assert np.array_equal(u32(out.scales.cpu().numpy()), u32(s))


# Every non-NaN E4M3 code in every block, with block scales on both sides of
# the block-table decode's fast range [2^-60, 2^60] (0, subnormal, the
# boundaries, huge): exercises the per-block table path and every fallback
# (zero/subnormal codes, extreme scales) of K3 and K4 against the oracle.
_VALID = np.array([c for c in range(256) if (c & 0x7F) != 0x7F], np.uint8)
_SCALES = np.array([0.0, 2.0 ** -60, 2.0 ** 60, 2.0 ** -61, 2.0 ** 61, 1e-40, 1e-30, 1e30, 1e37,
                    3.0, 0.125, 1.7e-5], np.float32)


def _all_code_blocks(rng, nblk):
    codes = np.concatenate([rng.permutation(_VALID)[:128] for _ in range(nblk)])
    scales = rng.choice(_SCALES, nblk).astype(np.float32)
    normal = rng.random(nblk) < 0.5
    scales[normal] = np.abs(rng.standard_normal(normal.sum())).astype(np.float32) * 10.0 ** rng.uniform(
        -8, 8, normal.sum()).astype(np.float32)
    return codes, scales


@pytest.mark.parametrize("world", [2, 4, 8])
def test_reduce_every_code_and_extreme_scales(cuda, world):
    rng = np.random.default_rng(100 + world)
    pieces = [_all_code_blocks(rng, 64) for _ in range(world)]
    oc, os_ = O.allreduce_decomposed([c for c, _ in pieces], [s for _, s in pieces])
    same(A.allreduce_simulated([fp8q(c, s, cuda) for c, s in pieces]), oc, os_)


def test_accumulate_every_code_and_extreme_scales(cuda):
    rng = np.random.default_rng(5)
    codes, scales = _all_code_blocks(rng, 64)
    local = (rng.standard_normal(codes.size) *
             np.repeat(10.0 ** rng.uniform(-30, 30, 64), 128)).astype(np.float32)
    local[rng.random(codes.size) < 0.05] = 0.0
    oc, os_ = O.local_accumulate(codes, scales, local)
    same(A.local_accumulate(fp8q(codes, scales, cuda), t(local, cuda)), oc, os_)


def test_nan_codes_abort_like_the_reference(cuda):
    rng = np.random.default_rng(9)
    codes, scales = _all_code_blocks(rng, 8)
    scales[:] = 1.0
    codes[300] = 0x7F  # NaN code in block 2
    with pytest.raises(O.OracleError) as ref:
        O.allreduce_decomposed([codes, codes], [scales, scales])
    with pytest.raises(A.ProtocolError) as got:
        A.allreduce_simulated([fp8q(codes, scales, cuda)] * 2)
    assert str(got.value) == ref.value.args[-1]
    local = np.zeros(codes.size, np.float32)
    with pytest.raises(O.OracleError) as ref:
        O.local_accumulate(codes, scales, local)
    with pytest.raises(A.InvalidArgument) as got:
        A.local_accumulate(fp8q(codes, scales, cuda), t(local, cuda))
    assert str(got.value) == ref.value.args[-1]


@pytest.mark.parametrize("n,world", [(512, 2), (513, 3), (1000, 8), (148 * 8 * 512 * 2 + 384, 4),
                                     ((1 << 22) + 300, 7), (1 << 21, 1)])
def test_reduce_pipeline_sizes(cuda, n, world):
    """K4's cp.async-ring kernel (whole 512-element warp-groups, several
    grid-stride rounds) plus its ragged tail, against the oracle."""
    rng = np.random.default_rng(n + world)
    codes, scales = [], []
    for _ in range(world):
        mag = np.repeat(10.0 ** rng.uniform(-6, 2, (n + 127) // 128), 128)[:n]
        c, s = O.quantize((rng.standard_normal(n) * mag).astype(np.float32), 8, 128, O.FP8)
        codes.append(c)
        scales.append(s)
    oc, os_ = O.allreduce_decomposed(codes, scales)
    same(A.allreduce_simulated([fp8q(c, s, cuda) for c, s in zip(codes, scales)]), oc, os_)


@pytest.mark.parametrize("world", [2, 5, 8])
def test_reduce_unaligned_scale_pointers(cuda, world):
    """The owner reduces a slice of its own gradient (chunk start = any block
    index), so piece scale pointers are only 4-byte aligned."""
    from paper_2605_00539_b200 import _lib as L
    rng = np.random.default_rng(40 + world)
    n = 128 * 1000
    codes, scales = [], []
    for _ in range(world):
        c, s = O.quantize((rng.standard_normal(n) * 1e-3).astype(np.float32), 8, 128, O.FP8)
        codes.append(c)
        scales.append(s)
    for skip in (1, 3):
        lo = skip * 128
        oc, os_ = O.allreduce_decomposed([c[lo:] for c in codes], [s[skip:] for s in scales])
        dc = [torch.from_numpy(c).to(cuda) for c in codes]
        ds = [torch.from_numpy(s).to(cuda) for s in scales]
        out_c = torch.empty(n - lo, dtype=torch.uint8, device=cuda)
        out_s = torch.empty(n // 128 - skip, dtype=torch.float32, device=cuda)
        err = A.ErrorRecord(cuda).reset()
        L.check(L.lib.agq_fp8_reduce_requant(
            world, L.ptr_array([c[lo:].data_ptr() for c in dc]),
            L.ptr_array([s[skip:].data_ptr() for s in ds]), n - lo, 128, 1,
            L.ptr_array([out_c.data_ptr()]), L.ptr_array([out_s.data_ptr()]), err.ptr,
            torch.cuda.current_stream().cuda_stream))
        L.errors_message(err.read(), L.AGQ_OP_ALLREDUCE)
        assert np.array_equal(out_c.cpu().numpy(), oc)
        assert np.array_equal(u32(out_s.cpu().numpy()), u32(os_))


def test_accumulate_validates_main_first(cuda):
    """local_accumulate dequantizes main first, so validate(main) runs before
    anything touches the data (collective.hpp:135 -> quantize.hpp:157-176)."""
    mc, ms = O.quantize(np.ones(300, np.float32), 8, 128, O.FP8)
    g = t(np.zeros(300, np.float32), cuda)
    bad = fp8q(mc, ms[:2], cuda)  # 3 blocks, 2 scales
    with pytest.raises(A.InvalidArgument, match="wrong number of scales"):
        A.local_accumulate(bad, g)
    q = fp8q(mc, ms, cuda)
    q.bit_width = 7
    with pytest.raises(A.InvalidArgument, match="fp8_e4m3 requires bit_width 8"):
        A.local_accumulate(q, g)
    q = fp8q(mc, ms, cuda)
    q.scales[1] = -2.0
    with pytest.raises(A.InvalidArgument, match="bad scale at block 1$"):
        A.local_accumulate(q, g)


@pytest.mark.parametrize("world", [3, 8, 12])
def test_allreduce_bad_scale_reports_lowest_worker(cuda, world):
    """check_workers validates the workers in order (collective.hpp:158-168):
    the error names the lowest bad block of the LOWEST worker with one, not
    the lowest bad block over all workers."""
    rng = np.random.default_rng(world)
    n = 8192 * 2 + 300
    mains = []
    for r in range(world):
        c, s = O.quantize(rng.standard_normal(n).astype(np.float32), 8, 128, O.FP8)
        if r == 1:
            s[100] = -1.0
            s[40] = np.nan
        if r == world - 1:
            s[3] = -0.5
        mains.append(fp8q(c, s, cuda))
    with pytest.raises(A.InvalidArgument, match="bad scale at block 40$"):
        A.allreduce_simulated(mains)
