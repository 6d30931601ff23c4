"""Activation / local-gradient buffers at 16-byte (but not 32-byte) and
32-byte offsets inside larger allocations. The warp kernels move each lane's
row with 256-bit accesses, so a 16-byte aligned buffer must take the generic
path and a 32-byte aligned one the fast path; either way the results are
bit-identical to the oracle (quantize.hpp:78-189, collective.hpp:128-147)."""
import numpy as np
import pytest
import torch

import oracle_ffi as O
import paper_2605_00539_b200 as A

pytestmark = pytest.mark.gpu
CODECS = [(A.CodecKind.SymmetricLinear, b) for b in (4, 5, 6, 7, 8)] + \
         [(A.CodecKind.Fp4E2M1, 4), (A.CodecKind.Fp8E4M3, 8)]
# (dtype, element offset): byte offset 16 (fast path refused) or 32 (taken)
OFFSETS = [(torch.bfloat16, 8), (torch.float32, 4), (torch.bfloat16, 16), (torch.float32, 8)]


def u32(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def at_offset(x: np.ndarray, dtype, off, dev):
    """x copied into base[off:] of a fresh allocation (returns the slice)."""
    base = torch.zeros(x.size + off, dtype=dtype, device=dev)
    view = base[off:]
    view.copy_(torch.from_numpy(x).to(dev).to(dtype))
    return view


def empty_at_offset(n, dtype, off, dev):
    return torch.empty(n + off, dtype=dtype, device=dev)[off:]


def inputs(n, seed, bf16):
    rng = np.random.default_rng(seed)
    x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3, (n + 127) // 128).repeat(128)[:n])
    x = x.astype(np.float32)
    x[rng.integers(0, n, n // 40)] = 0.0
    return O.bf16_round(x) if bf16 else x


@pytest.mark.parametrize("dtype,off", OFFSETS)
def test_quantize_dequantize_at_offsets(cuda, dtype, off):
    n = 3 * 8192 + 133
    x = inputs(n, off, dtype == torch.bfloat16)
    xt = at_offset(x, dtype, off, cuda)
    assert xt.data_ptr() % 32 == (off * xt.element_size()) % 32
    for kind, bits in CODECS:
        c, s = O.quantize(x, bits, 128, int(kind))
        q = A.quantize_blockwise(xt, bits, 128, kind)
        assert np.array_equal(q.codes.cpu().numpy(), O.pack(c, bits))
        assert np.array_equal(u32(q.scales.cpu().numpy()), u32(s))
        ref = O.dequantize(c, s, bits, 128, int(kind))
        out = empty_at_offset(n, dtype, off, cuda)
        A.dequantize_blockwise(q, dtype, out=out)
        want = O.bf16_round(ref) if dtype == torch.bfloat16 else ref
        assert np.array_equal(u32(out.float().cpu().numpy()), u32(want)), (kind, bits)


@pytest.mark.parametrize("off", [8, 16])
def test_roundtrip_and_grouped_at_offsets(cuda, off):
    n = 2 * 8192 + 64
    x = inputs(n, 100 + off, True)
    xt = at_offset(x, torch.bfloat16, off, cuda)
    c, s = O.quantize(x, 4, 128)
    want = O.bf16_round(O.dequantize(c, s, 4))
    q, y = A.quantize_roundtrip(xt, 4)
    assert np.array_equal(q.codes.cpu().numpy(), O.pack(c, 4))
    assert np.array_equal(u32(y.float().cpu().numpy()), u32(want))
    # a group mixing an offset tensor with an aligned one
    x2 = inputs(8192, 7, True)
    qs = A.quantize_grouped([xt, at_offset(x2, torch.bfloat16, 0, cuda)], 4)
    assert np.array_equal(qs[0].codes.cpu().numpy(), O.pack(c, 4))
    outs = [empty_at_offset(n, torch.bfloat16, off, cuda),
            empty_at_offset(8192, torch.bfloat16, 0, cuda)]
    A.dequantize_grouped(qs, torch.bfloat16, outs=outs)
    assert np.array_equal(u32(outs[0].float().cpu().numpy()), u32(want))
    c2, s2 = O.quantize(x2, 4, 128)
    assert np.array_equal(u32(outs[1].float().cpu().numpy()),
                          u32(O.bf16_round(O.dequantize(c2, s2, 4))))


@pytest.mark.parametrize("dtype,off", OFFSETS)
def test_accumulate_local_at_offsets(cuda, dtype, off):
    n = 4 * 512 * 37 + 128
    g = inputs(n, 3, False) * np.float32(1e-3)
    loc = inputs(n, 4 + off, dtype == torch.bfloat16) * np.float32(1e-3)
    loc = O.bf16_round(loc) if dtype == torch.bfloat16 else loc
    mc, ms = O.quantize(g, 8, 128, int(A.CodecKind.Fp8E4M3))
    main = A.QuantizedTensor(torch.from_numpy(mc).to(cuda), torch.from_numpy(ms).to(cuda), 8, 128,
                             (n,), A.CodecKind.Fp8E4M3, packed=False)
    lt = at_offset(loc, dtype, off, cuda)
    out = A.local_accumulate(main, lt)
    oc, os_ = O.local_accumulate(mc, ms, loc, 0)
    assert np.array_equal(out.codes.cpu().numpy(), oc)
    assert np.array_equal(u32(out.scales.cpu().numpy()), u32(os_))
