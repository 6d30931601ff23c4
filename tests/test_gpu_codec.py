"""GPU parity of the L1 block codec (K1 quantize+pack, K2 unpack+dequantize)
against the reference: the golden fixture made by the reference itself, the
C oracle on seeded inputs, and exhaustive element classes run ON the B200.
Bit-exact: codes, scales, packed bytes, FP32 dequantized values."""
import numpy as np
import pytest
import torch

import oracle_ffi as O
import paper_2605_00539_b200 as A

pytestmark = pytest.mark.gpu
CODECS = [(A.CodecKind.SymmetricLinear, b) for b in (4, 5, 6, 7, 8)] + \
         [(A.CodecKind.Fp4E2M1, 4), (A.CodecKind.Fp8E4M3, 8)]


def t(x, dev, dtype=torch.float32):
    return torch.from_numpy(np.ascontiguousarray(x)).to(dev).to(dtype)


def u32(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def check_q(q, codes, scales, bits):
    got_s = q.scales.cpu().numpy()
    assert np.array_equal(u32(got_s), u32(scales))
    if q.packed:
        assert np.array_equal(q.codes.cpu().numpy(), O.pack(codes, bits))
    else:
        assert np.array_equal(q.codes.cpu().numpy(), codes)


@pytest.mark.parametrize("name", ["x_cli", "x_cli_bf16", "x_codec", "x_ragged"])
@pytest.mark.parametrize("block", [128, 16, 1000])
def test_golden(cuda, golden, name, block):
    x = golden[name]
    for kind, bits in CODECS:
        key = f"{name}_c{int(kind)}_b{bits}_k{block}"
        for packed in (True, False):
            q = A.quantize_blockwise(t(x, cuda), bits, block, kind, packed=packed)
            check_q(q, golden[key + "_codes"], golden[key + "_scales"], bits)
            d = A.dequantize_blockwise(q).cpu().numpy()
            assert np.array_equal(u32(d), u32(golden[key + "_deq"])), key
        if name == "x_cli_bf16":  # BF16 input path gives the same codes
            q = A.quantize_blockwise(t(x, cuda, torch.bfloat16), bits, block, kind)
            check_q(q, golden[key + "_codes"], golden[key + "_scales"], bits)
            d = A.dequantize_blockwise(q, torch.bfloat16).float().cpu().numpy()
            assert np.array_equal(u32(d), u32(O.bf16_round(golden[key + "_deq"]))), key


def _random_case(rng, n, bf16):
    x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3)).astype(np.float32)
    x[rng.integers(0, n, size=max(1, n // 50))] = 0.0
    nb = (n + 127) // 128
    if nb > 3:  # per-block magnitudes, zero blocks, extreme-scale blocks
        scale = 10.0 ** rng.uniform(-6, 6, size=nb)
        scale[rng.integers(0, nb, size=max(1, nb // 20))] = 0.0
        scale[1] = 1e-25
        scale[2] = 1e25
        x = (x * np.repeat(scale, 128)[:n]).astype(np.float32)
    return O.bf16_round(x) if bf16 else x


@pytest.mark.parametrize("n", [1, 127, 128, 8191, 8192, 8192 * 3 + 129, 100003])
@pytest.mark.parametrize("bf16", [True, False])
def test_random_vs_oracle(cuda, n, bf16):
    rng = np.random.default_rng(n + bf16)
    x = _random_case(rng, n, bf16)
    xt = t(x, cuda, torch.bfloat16 if bf16 else torch.float32)
    for kind, bits in CODECS:
        c, s = O.quantize(x, bits, 128, int(kind))
        for packed in (True, False):
            q = A.quantize_blockwise(xt, bits, 128, kind, packed=packed)
            check_q(q, c, s, bits)
            d = A.dequantize_blockwise(q).cpu().numpy()
            assert np.array_equal(u32(d), u32(O.dequantize(c, s, bits, 128, int(kind))))
            db = A.dequantize_blockwise(q, torch.bfloat16).float().cpu().numpy()
            assert np.array_equal(u32(db), u32(O.bf16_round(O.dequantize(c, s, bits, 128, int(kind)))))


def test_misaligned_pointers_take_generic_path(cuda):
    rng = np.random.default_rng(9)
    x = _random_case(rng, 3 * 8192 + 5, True)
    base = t(np.concatenate([[0.0], x]).astype(np.float32), cuda, torch.bfloat16)
    xt = base[1:]  # 2-byte offset: not 16-byte aligned
    for kind, bits in CODECS:
        c, s = O.quantize(x, bits, 128, int(kind))
        check_q(A.quantize_blockwise(xt, bits, 128, kind), c, s, bits)


def test_c1_full_size(cuda):
    """Config C1: 4096x4096 BF16, INT4 block 128, reference RNG inputs."""
    if O.ref is None:
        pytest.skip("reference RNG lib absent")
    x = O.bf16_round(O.ref_normal(1, 0x1D, 0, 4096 * 4096))
    q = A.quantize_blockwise(t(x, cuda, torch.bfloat16), 4, 128)
    c, s = O.quantize(x, 4, 128)
    check_q(q, c, s, 4)
    d = A.dequantize_blockwise(q, torch.bfloat16).float().cpu().numpy()
    assert np.array_equal(u32(d), u32(O.bf16_round(O.dequantize(c, s, 4))))


def test_nonfinite_reports_lowest_block(cuda):
    x = np.random.default_rng(8).standard_normal(300).astype(np.float32)
    x[170] = np.inf
    with pytest.raises(A.InvalidArgument, match="non-finite input element in block 1"):
        A.quantize_blockwise(t(x, cuda), 4, 128)
    y = np.random.default_rng(1).standard_normal(8192 * 4).astype(np.float32)
    y[8192 * 2 + 300] = np.nan
    y[8192 * 3 + 5] = -np.inf
    with pytest.raises(A.InvalidArgument, match="block 130$"):
        A.quantize_blockwise(t(y, cuda, torch.bfloat16), 5, 128)


def test_validate_errors(cuda):
    q = A.quantize_blockwise(t(np.ones(300, np.float32), cuda), 5, 128, packed=False)
    q.codes[7] = 200
    with pytest.raises(A.InvalidArgument, match="code out of range at 7"):
        A.dequantize_blockwise(q)
    q = A.quantize_blockwise(t(np.ones(300, np.float32), cuda), 5, 128)
    q.scales[2] = -1.0
    with pytest.raises(A.InvalidArgument, match="bad scale at block 2"):
        A.dequantize_blockwise(q)


def test_edge_sizes(cuda):
    for n in (0, 1, 2, 3):
        x = np.arange(n, dtype=np.float32) - 1.0
        for kind, bits in CODECS:
            q = A.quantize_blockwise(t(x, cuda), bits, 2, kind)
            c, s = O.quantize(x, bits, 2, int(kind)) if n else (np.zeros(0, np.uint8), np.zeros(0, np.float32))
            check_q(q, c, s, bits)


def test_grouped_equals_single(cuda):
    rng = np.random.default_rng(2)
    xs = [t(_random_case(rng, n, True), cuda, torch.bfloat16) for n in (8192 * 5, 8192 * 2 + 77, 300)]
    for bits in (4, 5, 6, 7, 8):
        qs = A.quantize_grouped(xs, bits)
        for x, q in zip(xs, qs):
            r = A.quantize_blockwise(x, bits)
            assert torch.equal(q.codes, r.codes) and torch.equal(q.scales, r.scales)
        outs = A.dequantize_grouped(qs, torch.bfloat16)
        for q, o in zip(qs, outs):
            assert torch.equal(o.reshape(-1), A.dequantize_blockwise(q, torch.bfloat16).reshape(-1))


def test_pack_unpack_device(cuda):
    rng = np.random.default_rng(991)
    for bits in range(4, 9):
        for n in (1, 7, 8, 129, 1000, 100001):
            codes = rng.integers(0, 1 << bits, size=n).astype(np.uint8)
            p = A.pack_codes(t(codes, cuda, torch.uint8), bits)
            assert np.array_equal(p.cpu().numpy(), O.pack(codes, bits))
            u = A.unpack_codes(p, bits, n)
            assert np.array_equal(u.cpu().numpy(), codes)


def _bf16_domain_blocks(a_exp=0):
    """Every BF16 x with |x| <= a for every BF16 mantissa a in [1,2) (scaled
    by 2^a_exp): blocks of 128 = [a, x_1 .. x_127]."""
    mags = (np.arange(0x8000, dtype=np.uint32) << 16).view(np.float32)
    rows = []
    for am in range(128):
        a1 = np.array([(0x3F80 | am) << 16], np.uint32).view(np.float32)[0]
        a = np.float32(np.ldexp(np.float64(a1), a_exp))
        xs = mags[mags <= a]
        xs = np.concatenate([xs, -xs])
        pad = (-len(xs)) % 127
        xs = np.concatenate([xs, np.zeros(pad, np.float32)]).reshape(-1, 127)
        blk = np.concatenate([np.full((xs.shape[0], 1), a, np.float32), xs], axis=1)
        rows.append(blk.reshape(-1))
    return np.concatenate(rows).astype(np.float32)


@pytest.mark.parametrize("a_exp", [0, -59, 59])
def test_exhaustive_bf16_classes_on_device(cuda, a_exp):
    """Same domain as tests/cpp/numerics_check.cpp, run through the kernels."""
    x = _bf16_domain_blocks(a_exp)
    for bf16 in (True, False):
        xt = t(x, cuda, torch.bfloat16 if bf16 else torch.float32)
        for kind, bits in CODECS:
            c, s = O.quantize(x, bits, 128, int(kind))
            q = A.quantize_blockwise(xt, bits, 128, kind, packed=False)
            got = q.codes.cpu().numpy()
            bad = np.nonzero(got != c)[0]
            assert bad.size == 0, (kind, bits, bf16, bad[:5], x[bad[:5]])


def test_exhaustive_dequant_bf16_scales_on_device(cuda):
    """Every code x every BF16 scale in [2^-62, 2^62] (+ extremes)."""
    exps = np.arange(-62, 62)
    sm = np.arange(128, dtype=np.uint32)
    base = ((0x3F80 | sm) << 16).view(np.float32)
    scales = (base[None, :] * np.ldexp(1.0, exps)[:, None]).astype(np.float32).reshape(-1)
    scales = np.concatenate([scales, np.array([0.0, 1e-40, 3e38, 1.5e-45], np.float32)])
    for kind, bits in CODECS:
        ncode = 1 << bits
        codes = np.tile(np.arange(ncode, dtype=np.uint8), (scales.size, (128 + ncode - 1) // ncode))[:, :128]
        codes = np.ascontiguousarray(codes.reshape(-1))
        if kind == A.CodecKind.Fp8E4M3:
            codes[(codes & 0x7F) == 0x7F] = 0
        q = A.QuantizedTensor(t(codes, cuda, torch.uint8), t(scales, cuda), bits, 128,
                              (codes.size,), kind, packed=False)
        d = A.dequantize_blockwise(q).cpu().numpy()
        want = O.dequantize(codes, scales, bits, 128, int(kind))
        assert np.array_equal(u32(d), u32(want)), (kind, bits)


def test_fp8_hardware_cvt_matches_rne(cuda):
    """cvt.rn.satfinite.e4m3x2 (used by the gradient requant) == fp8_encode's
    RNE: fp8 quantize of blocks anchored at 448 = encode of the value itself."""
    rng = np.random.default_rng(0)
    v = np.concatenate([rng.uniform(0, 448, 2_000_000), rng.uniform(0, 2 ** -5, 500_000)]).astype(np.float32)
    v = np.concatenate([v, -v])
    pad = (-v.size) % 127
    v = np.concatenate([v, np.zeros(pad, np.float32)]).reshape(-1, 127)
    x = np.concatenate([np.full((v.shape[0], 1), 448.0, np.float32), v], axis=1).reshape(-1)
    q = A.quantize_blockwise(t(x, cuda), 8, 128, A.CodecKind.Fp8E4M3, packed=False)
    c, _ = O.quantize(x, 8, 128, O.FP8)
    assert np.array_equal(q.codes.cpu().numpy(), c)


def test_launches_are_counted(cuda):
    n0 = A.launch_count()
    A.quantize_blockwise(t(np.ones(8192, np.float32), cuda, torch.bfloat16), 4)
    assert A.launch_count() > n0


def test_c2_layer_store_sampled(cuda):
    """Config C2: one LLaMA-8B block's stored activations (T=16384 tokens)
    under every 8-stage DBCA policy through ActivationStore (grouped
    launches); sampled blocks of every tensor bit-exact vs the oracle, and
    the reconstruction is the oracle's BF16-rounded dequantization."""
    T = 4 * 4096
    g = torch.Generator(device=cuda).manual_seed(5)
    acts = {"norm1_input": torch.randn(T * 4096, device=cuda, generator=g).to(torch.bfloat16),
            "norm2_input": torch.randn(T * 4096, device=cuda, generator=g).to(torch.bfloat16),
            "outproj_input": (torch.randn(T * 4096, device=cuda, generator=g) * 0.5).to(torch.bfloat16),
            "silu_gate": (torch.randn(T * 14336, device=cuda, generator=g) * 4).to(torch.bfloat16),
            "silu_value": torch.randn(T * 14336, device=cuda, generator=g).to(torch.bfloat16),
            "q": torch.randn(T * 4096, device=cuda, generator=g).to(torch.bfloat16)}
    plan = A.plan_bit_widths(A.PipelineConfig(8, 16, 2))
    rng = np.random.default_rng(2)
    for stage in range(1, 9):
        store = A.ActivationStore(A.stage_policy(plan, stage))
        store.store(acts)
        bits = plan.stages[stage - 1].assigned_bits
        assert store.entries["q"] is acts["q"]  # attention stays full precision
        for name in ("norm1_input", "silu_gate", "outproj_input"):
            q = store.entries[name]
            assert q.bit_width == bits and q.packed
            back = store.read(name)
            for b in rng.integers(0, acts[name].numel() // 128, 6):
                x = acts[name][b * 128:(b + 1) * 128].float().cpu().numpy()
                c, s = O.quantize(x, bits, 128)
                got = q.codes[b * 16 * bits:(b + 1) * 16 * bits].cpu().numpy()
                assert np.array_equal(got, O.pack(c, bits))
                want = O.bf16_round(O.dequantize(c, s, bits))
                assert np.array_equal(u32(back[b * 128:(b + 1) * 128].float().cpu().numpy()), u32(want))


@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_dequant_fp8_fp32_scales(cuda, out_dtype):
    """FP8 codes with FP32 (non-BF16) block scales — the FP8 gradient case:
    every code in every block, random FP32 scales plus the table path's range
    edges, vs the oracle's (float)(unit * (double)s)."""
    rng = np.random.default_rng(3)
    nblk = 4096
    codes = np.concatenate([rng.permutation(256).astype(np.uint8)[:128] for _ in range(nblk)])
    scales = (rng.random(nblk) * 10.0 ** rng.uniform(-20, 20, nblk)).astype(np.float32)
    scales[:8] = np.array([0.0, 2.0 ** -60, 2.0 ** 60, 2.0 ** -61, 2.0 ** 61, 1e-40, 3e38, 1.0],
                          np.float32)
    nz = rng.random(codes.size) < 0.001  # some rows with NaN codes too
    codes[nz] = 0x7F
    q = A.QuantizedTensor(t(codes, cuda, torch.uint8), t(scales, cuda), 8, 128, (codes.size,),
                          A.CodecKind.Fp8E4M3, packed=False)
    d = A.dequantize_blockwise(q, out_dtype=out_dtype).float().cpu().numpy()
    want = O.dequantize(codes, scales, 8, 128, O.FP8)
    if out_dtype == torch.bfloat16:
        want = O.bf16_round(want)
    assert np.array_equal(u32(d), u32(want))


@pytest.mark.parametrize("bits", [4, 5, 6, 7, 8])
def test_roundtrip_fused_equals_two_calls(cuda, bits):
    """agq_quantize_roundtrip (one fused pass for SymmetricLinear BF16 at
    block 128) = quantize_blockwise then dequantize_blockwise, bit for bit:
    whole tiles, a ragged tail, zero and extreme blocks."""
    rng = np.random.default_rng(bits)
    x = _random_case(rng, 8192 * 5 + 300, True)
    x[128:256] = 0.0
    x[1024:1152] *= 2.0 ** 70
    xt = t(x, cuda, torch.bfloat16)
    q, y = A.quantize_roundtrip(xt, bits)
    r = A.quantize_blockwise(xt, bits)
    assert torch.equal(q.codes, r.codes) and torch.equal(q.scales, r.scales)
    assert torch.equal(y, A.dequantize_blockwise(r, torch.bfloat16))
    c, s = O.quantize(xt.float().cpu().numpy(), bits, 128)
    assert np.array_equal(u32(y.float().cpu().numpy()), u32(O.bf16_round(O.dequantize(c, s, bits))))
    # other codecs / dtypes go through the two-call path, same results
    for kind, b in ((A.CodecKind.Fp8E4M3, 8), (A.CodecKind.Fp4E2M1, 4)):
        q2, y2 = A.quantize_roundtrip(xt.float(), b, 128, kind)
        r2 = A.quantize_blockwise(xt.float(), b, 128, kind)
        assert torch.equal(q2.codes, r2.codes) and torch.equal(y2, A.dequantize_blockwise(r2))
    d = A.roundtrip_relative_delta(xt.float(), bits)
    xd = xt.float().double().cpu()
    want = torch.where(xd == 0, torch.zeros_like(xd),
                       (torch.from_numpy(O.dequantize(c, s, bits)).double() - xd) / xd)
    assert torch.equal(d.cpu(), want)


def test_error_record_reset_skipped_after_clean_read(cuda):
    """A record read back clean is not reset again (one kernel launch saved
    per checked call); handing out its pointer makes it dirty again."""
    x = torch.randn(8192, device=cuda)
    err = A.ErrorRecord(cuda)
    A.quantize_blockwise(x, 4, errors=err)  # checked call: reset, kernel, clean read
    assert err._clean
    n0 = A.launch_count()
    err.reset()
    assert A.launch_count() == n0  # skipped
    _ = err.ptr
    err.reset()
    assert A.launch_count() == n0 + 1
    bad = x.clone()
    bad[5] = float("nan")
    with pytest.raises(A.InvalidArgument):
        A.quantize_blockwise(bad, 4, errors=err)
    assert not err._clean  # an error was read: the next use resets
