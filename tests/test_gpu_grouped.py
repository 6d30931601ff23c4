"""Grouped launches over a whole pipeline stage (layers.hpp:266-301 stored
set of every layer, dbca.hpp:172-177 stage width): any number of tensors in
one call (one launch per 8 segments), equal to the single-tensor path, and the
reference's validate errors (quantize.hpp:157-179) from grouped dequantize,
reported for the first failing tensor with its own local index."""
import numpy as np
import pytest
import torch

import oracle_ffi as O
import paper_2605_00539_b200 as A

pytestmark = pytest.mark.gpu


def _layers(dev, nlayers, T, seed):
    g = torch.Generator(device=dev).manual_seed(seed)
    out = []
    for _ in range(nlayers):
        d = {"norm1_input": T * 512, "norm2_input": T * 512, "outproj_input": T * 512,
             "silu_gate": T * 1792, "silu_value": T * 1792, "q": T * 512}
        out.append({k: torch.randn(n, device=dev, generator=g).to(torch.bfloat16)
                    for k, n in d.items()})
    return out


def test_stage_store_4_layers_20_tensors_one_call(cuda):
    layers = _layers(cuda, 4, 256, 1)
    plan = A.plan_bit_widths(A.PipelineConfig(8, 16, 2))
    for stage in (1, 5, 8):
        store = A.StageActivationStore(A.stage_policy(plan, stage))
        n0 = A.launch_count()
        store.store(layers)
        # 20 tensors, one width: three launches of up to 8 segments, plus the
        # error-record reset (a kernel, so the call is graph-capturable)
        assert A.launch_count() - n0 == 3 + 1
        bits = plan.stages[stage - 1].assigned_bits
        back = store.read_all()
        for li, d in enumerate(layers):
            assert store.layers[li]["q"] is d["q"]
            for name in ("norm1_input", "norm2_input", "outproj_input", "silu_gate", "silu_value"):
                q = store.layers[li][name]
                r = A.quantize_blockwise(d[name], bits)
                assert torch.equal(q.codes, r.codes) and torch.equal(q.scales, r.scales)
                ref = A.dequantize_blockwise(r, torch.bfloat16)
                assert torch.equal(back[li][name], ref)
                assert torch.equal(store.read(li, name), ref)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_grouped_many_tensors_ragged(cuda, dtype):
    rng = np.random.default_rng(7)
    sizes = [int(s) for s in rng.integers(1, 40000, 45)] + [8192 * 3, 1024, 128 * 9 + 5]
    xs = [torch.from_numpy(rng.standard_normal(n).astype(np.float32)).to(cuda).to(dtype)
          for n in sizes]
    for bits in (4, 7):
        qs = A.quantize_grouped(xs, bits)
        outs = A.dequantize_grouped(qs, torch.float32)
        for x, q, o in zip(xs, qs, outs):
            c, s = O.quantize(x.float().cpu().numpy(), bits, 128)
            assert np.array_equal(q.codes.cpu().numpy(), O.pack(c, bits))
            assert np.array_equal(q.scales.cpu().numpy().view(np.uint32), s.view(np.uint32))
            assert np.array_equal(o.cpu().numpy().view(np.uint32),
                                  O.dequantize(c, s, bits).view(np.uint32))


def test_grouped_dequant_validates_like_the_reference(cuda):
    rng = np.random.default_rng(9)
    sizes = [8192 * 2, 300, 8192 + 77, 5000]
    xs = [torch.from_numpy(rng.standard_normal(n).astype(np.float32)).to(cuda) for n in sizes]
    qs = A.quantize_grouped(xs, 5)
    qs[2].scales[3] = -1.0  # segment 2, local block 3
    qs[3].scales[1] = float("nan")
    with pytest.raises(A.InvalidArgument, match="bad scale at block 3$") as e:
        A.dequantize_grouped(qs)
    assert e.value.segment == 2
    qs[1].scales[0] = float("inf")  # an earlier tensor fails first
    with pytest.raises(A.InvalidArgument, match="bad scale at block 0$") as e:
        A.dequantize_grouped(qs)
    assert e.value.segment == 1
    qs[2].scales[3] = 1.0
    qs[1].scales[0] = 1.0
    with pytest.raises(A.InvalidArgument, match="bad scale at block 1$") as e:
        A.dequantize_grouped(qs)
    assert e.value.segment == 3
    # validate off: no error, values computed
    A.dequantize_grouped(qs, validate=False, check=False)


def test_grouped_nonfinite_input_reports_local_block(cuda):
    xs = [torch.randn(n, device=cuda) for n in (8192, 8192 * 2 + 300, 4096)]
    xs[1][8192 + 129] = float("inf")
    with pytest.raises(A.InvalidArgument, match="non-finite input element in block 65$") as e:
        A.quantize_grouped(xs, 4)
    assert e.value.segment == 1
