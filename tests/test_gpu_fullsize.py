"""Full-size parity of the headline activation config (C2) against the
reference itself (oracle/_ref: the unmodified reference headers compiled
as-is): all five stored tensors of one LLaMA-8B block at T = 16,384 tokens
(671,088,640 elements, the reference RNG's bytes, BF16-valued), at every
DBCA width 4..8, through the grouped launch the bench times. Packed codes,
scales, FP32 reconstruction bit-exact; BF16 reconstruction = its RNE.
Every tensor is <= 2^28 elements, so the comparison is complete, not sampled
(quantize.hpp:78-189, tensor_io.hpp:63-80)."""
import os

import numpy as np
import pytest
import torch

import oracle_ffi as O
import paper_2605_00539_b200 as A
from paper_2605_00539_b200.inputs import materialize_parallel

pytestmark = pytest.mark.gpu

T = 4 * 4096
SIZES = [T * 4096] * 3 + [T * 14336] * 2  # norm1, norm2, out-proj inputs; SiLU gate, value
SCALES = (1.0, 1.0, 0.5, 4.0, 1.0)


def _threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def test_c2_full_tensors_every_width(cuda):
    if O.ref is None:
        pytest.skip("oracle/_ref not built")
    th = _threads()
    host = materialize_parallel(SIZES, 0, torch.bfloat16, scales=SCALES)
    xs = [h.to(cuda) for h in host]
    for b in (4, 5, 6, 7, 8):
        qs = A.quantize_grouped(xs, b)
        outs32 = A.dequantize_grouped(qs, torch.float32)
        outs16 = A.dequantize_grouped(qs, torch.bfloat16)
        for i, h in enumerate(host):
            xf = h.float().numpy()
            n = xf.size
            codes = np.empty(n, np.uint8)
            scales = np.empty(n // 128, np.float32)
            assert O.ref.ref_quantize_mt(O._p(xf), n, b, 128, 0, O._p(codes), O._p(scales), th) == 0
            packed = np.empty(n * b // 8 + 1, np.uint8)
            k = O.ref.ref_pack_codes(O._p(codes), n, b, O._p(packed))
            assert np.array_equal(qs[i].codes.cpu().numpy(), packed[:k]), (i, b, "codes")
            assert np.array_equal(qs[i].scales.cpu().numpy().view(np.uint32),
                                  scales.view(np.uint32)), (i, b, "scales")
            ref = np.empty(n, np.float32)
            assert O.ref.ref_dequantize_mt(O._p(codes), O._p(scales), n, b, 128, 0, O._p(ref),
                                           th) == 0
            rt = torch.from_numpy(ref).to(cuda)
            assert torch.equal(outs32[i].view(torch.int32), rt.view(torch.int32)), (i, b, "f32")
            assert torch.equal(outs16[i].view(torch.int16),
                               rt.to(torch.bfloat16).view(torch.int16)), (i, b, "bf16")
            del rt
        del qs, outs32, outs16
        torch.cuda.empty_cache()


def test_c1_reference_cli_bytes(cuda):
    """C1 on the reference CLI's own input (`--seed 1 --normal 16777216`,
    agq.cpp:47-65), FP32 and BF16-rounded, INT4 block 128: bit-exact against
    oracle/_ref."""
    if O.ref is None:
        pytest.skip("oracle/_ref not built")
    from paper_2605_00539_b200.inputs import materialize
    n = 4096 * 4096
    x = materialize(n, 1)
    assert np.array_equal(x.numpy().view(np.uint32), O.ref_normal(1, 0x1D, 0, n).view(np.uint32))
    th = _threads()
    for dt in (torch.float32, torch.bfloat16):
        xd = x.to(cuda).to(dt)
        xf = xd.float().cpu().numpy()
        q = A.quantize_blockwise(xd, 4)
        codes = np.empty(n, np.uint8)
        scales = np.empty(n // 128, np.float32)
        assert O.ref.ref_quantize_mt(O._p(xf), n, 4, 128, 0, O._p(codes), O._p(scales), th) == 0
        assert np.array_equal(q.codes.cpu().numpy(), O.pack(codes, 4, O.ref))
        assert np.array_equal(q.scales.cpu().numpy().view(np.uint32), scales.view(np.uint32))
        ref = np.empty(n, np.float32)
        assert O.ref.ref_dequantize_mt(O._p(codes), O._p(scales), n, 4, 128, 0, O._p(ref), th) == 0
        got = A.dequantize_blockwise(q).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
