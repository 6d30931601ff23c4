"""The C-ABI library loads, exports every symbol include/agq_cuda.h declares,
and its host-side logic (argument checks with the reference's messages, chunk
assignment, DBCA planner, error translation) matches the reference — no GPU
compute here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle_ffi as O
import paper_2605_00539_b200 as A
from paper_2605_00539_b200 import _lib as L

HDR = os.path.join(O.ROOT, "include", "agq_cuda.h")


def declared_symbols():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(agq_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 30
    lib = C.CDLL(L.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(L.EXPORTED)


@pytest.mark.parametrize("nbytes", [0, 17, 65536 + 3, (5 << 20) + 11])
def test_host_copy(nbytes):
    """agq_host_copy: the staging copy of the host pipelines (copy threads,
    streaming stores, ragged head/tail) — pure host code."""
    rng = np.random.default_rng(nbytes)
    src = rng.integers(0, 256, nbytes + 64, dtype=np.uint8)
    dst = np.zeros_like(src)
    # odd offsets: unaligned head and tail around the streaming body
    L.check(L.lib.agq_host_copy(dst.ctypes.data + 1, src.ctypes.data + 3, nbytes))
    assert np.array_equal(dst[1:1 + nbytes], src[3:3 + nbytes])
    assert not dst[0] and not dst[1 + nbytes:].any()
    if nbytes:
        assert L.lib.agq_host_copy(None, src.ctypes.data, nbytes) != 0


def test_library_is_sm100a_only():
    out = os.popen(f"cuobjdump --list-elf {L.LIB_PATH} 2>/dev/null").read()
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.parametrize("bits,block,codec,msg", [
    (3, 128, 0, "bit_width must be in [4, 8], got 3"),
    (9, 128, 0, "bit_width must be in [4, 8], got 9"),
    (4, 0, 0, "block_size must be >= 1"),
    (5, 128, 2, "fp8_e4m3 requires bit_width 8"),
    (5, 128, 1, "fp4_e2m1 requires bit_width 4"),
])
def test_codec_arg_errors(bits, block, codec, msg):
    with pytest.raises(A.InvalidArgument, match=re.escape(msg)):
        A.check_codec_args(bits, block, codec)


def test_chunk_assignment_matches_reference():
    assert A.ChunkAssignment.block_aligned(4096, 128, 4).ranges == \
        [(0, 1024), (1024, 2048), (2048, 3072), (3072, 4096)]
    assert A.ChunkAssignment.block_aligned(300, 128, 2).ranges == [(0, 256), (256, 300)]
    rng = np.random.default_rng(0)
    for _ in range(200):
        n, blk, w = int(rng.integers(0, 10 ** 7)), int(rng.integers(1, 300)), int(rng.integers(1, 17))
        r = np.zeros(2 * w, np.uint64)
        O.orc.oracle_chunk_assignment(n, blk, w, O._p(r))
        assert A.ChunkAssignment.block_aligned(n, blk, w).ranges == \
            [(int(r[2 * i]), int(r[2 * i + 1])) for i in range(w)]
    with pytest.raises(A.InvalidArgument, match="need at least one worker"):
        A.ChunkAssignment.block_aligned(10, 128, 0)


def test_planner_matches_oracle():
    for n in (1, 2, 3, 4, 5, 8, 12, 16):
        for mb in (2 * n, 2 * n + 3, 64):
            p = A.plan_bit_widths(A.PipelineConfig(n, mb, 2))
            c = (C.c_int * n)(); r = (C.c_double * n)(); a = (C.c_int * n)()
            assert O.orc.oracle_plan_bit_widths(n, mb, 2, c, r, a) == 0
            assert [s.stored_minibatches for s in p.stages] == list(c)
            assert [s.assigned_bits for s in p.stages] == list(a)
            assert [s.raw_bits for s in p.stages] == list(r)
    assert A.plan_bit_widths(A.PipelineConfig(4, 8, 2)).assigned() == [4, 5, 6, 8]
    for cfg, msg in (((4, 6, 2), "micro_batches >= 2 * n_stages"), ((4, 8, 3), "interleave"),
                     ((0, 8, 2), "n_stages must be >= 1")):
        with pytest.raises(A.InvalidArgument, match=re.escape(msg)):
            A.stored_activation_counts(A.PipelineConfig(*cfg))


def test_policy_and_checks():
    plan = A.plan_bit_widths(A.PipelineConfig(4, 8, 2))
    pol = A.stage_policy(plan, 2)                                 # test_dbca.cpp:105-112
    assert pol.at(A.LayerRole.RmsNorm).bit_width == 5
    assert pol.at(A.LayerRole.Attention).strategy == A.SaveStrategy.NoQuant
    with pytest.raises(A.InvalidArgument):
        A.stage_policy(plan, 9)
    chk = A.peak_memory_check(plan, 16.0)                         # :59-80
    assert chk.passed and chk.budget_bytes == 44.0
    assert [s["bytes"] for s in chk.stages] == [44.0, 45.0, 42.0, 40.0]
    reuse = A.plan_reuse_check(A.PipelineConfig(4, 8, 2), A.PipelineConfig(8, 16, 2))
    assert reuse["applied_bits"] == [4, 4, 4, 4, 4, 5, 6, 8] and reuse["pass"]
    assert reuse["uniform4_peak"] == 92.0


def test_error_translation_texts():
    h = L.AgqErrors(L.INT64_MAX, L.INT64_MAX, L.INT64_MAX, L.INT64_MAX, L.INT64_MAX, 0)
    L.errors_message(h, L.AGQ_OP_QUANTIZE)  # no error -> no raise
    h.nonfinite_block = 1
    with pytest.raises(A.InvalidArgument, match="non-finite input element in block 1"):
        L.errors_message(h, L.AGQ_OP_QUANTIZE)
    h = L.AgqErrors(L.INT64_MAX, 3, 7, L.INT64_MAX, L.INT64_MAX, 0)
    with pytest.raises(A.InvalidArgument, match="code out of range at 7"):
        L.errors_message(h, L.AGQ_OP_DEQUANTIZE)
    h = L.AgqErrors(2, L.INT64_MAX, L.INT64_MAX, 5, L.INT64_MAX, 0)
    with pytest.raises(A.InvalidArgument, match="non-finite local gradient element"):
        L.errors_message(h, L.AGQ_OP_ACCUMULATE)
    h = L.AgqErrors(L.INT64_MAX, L.INT64_MAX, L.INT64_MAX, L.INT64_MAX, 4, 0)
    with pytest.raises(A.ProtocolError, match="fp32 overflow during local reduce"):
        L.errors_message(h, L.AGQ_OP_ALLREDUCE)


def test_trace_matches_reference(golden):
    for world in (2, 4, 8):
        ev = A.decomposed_trace(1024, 128, world)
        ref = golden[f"ar{world}_trace"]
        assert len(ev) == len(ref)
        for e, r in zip(ev, ref):
            phase = {"all_to_all": 0, "all_gather": 1}[e.phase]
            assert (phase, e.sender, e.receiver, e.chunk_start, e.chunk_len, e.payload_bytes) == \
                tuple(int(v) for v in r)


@pytest.mark.parametrize("n,world", [(1024, 2), (1024, 4), (1024, 8), (300, 4), (128 * 7 + 5, 3), (64, 1)])
def test_naive_trace_matches_reference(n, world):
    """naive_trace == the MessageTrace of the reference's own
    allreduce_naive_fp8 (collective.hpp:356-421), empty chunks included."""
    rng = np.random.default_rng(n + world)
    codes, scales = [], []
    for _ in range(world):
        c, s = O.quantize(rng.standard_normal(n).astype(np.float32), 8, 128, O.FP8)
        codes.append(c)
        scales.append(s)
    ref = O.ref_allreduce(1, codes, scales)[3]
    ev = A.naive_trace(n, 128, world)
    assert len(ev) == len(ref)
    for e, r in zip(ev, ref):
        phase = {"all_to_all": 0, "all_gather": 1, "reduce_scatter": 2}[e.phase]
        assert (phase, e.sender, e.receiver, e.chunk_start, e.chunk_len, e.payload_bytes) == \
            tuple(int(v) for v in r)


def test_scalar_formats_match_oracle():
    for b in range(256):
        x = O.orc.oracle_fp8_decode(b)
        y = A.fp8_decode(b)
        assert (np.isnan(x) and np.isnan(y)) or x == y
        if not np.isnan(x):
            assert A.fp8_encode(x).byte == b
    rng = np.random.default_rng(4)
    for v in rng.standard_normal(3000) * 100:
        ov = C.c_int(0)
        assert A.fp8_encode(float(v)).byte == O.orc.oracle_fp8_encode(float(v), C.byref(ov))
        assert A.fp8_encode(float(v)).overflow == bool(ov.value)
        assert A.fp4_encode(float(v) / 20) == O.orc.oracle_fp4_encode(float(v) / 20)


def test_no_device_means_error_not_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    x = np.ones(16, np.float32)
    c = np.zeros(16, np.uint8)
    s = np.zeros(1, np.float32)
    st = L.lib.agq_quantize_host(x.ctypes.data, 16, 4, 128, 0, c.ctypes.data, s.ctypes.data)
    assert st == L.AGQ_ERR_CUDA


def test_fill_input_is_the_reference_rng():
    """agq_fill_input (host) = make_rng(seed, stream, index) +
    std::normal_distribution<float> of the reference (rng.hpp:9-28,
    agq.cpp:47-65), byte for byte; BF16 output = its RNE."""
    import torch
    from paper_2605_00539_b200.inputs import materialize, materialize_parallel
    if O.ref is None:
        pytest.skip("oracle/_ref not built")
    for seed, idx, n, std in [(0, 0, 4096, 1.0), (1, 0, 100003, 1.0), (7, 3, 5000, 1e-3),
                              (2**63 + 5, 1, 257, 4.0)]:
        a = materialize(n, seed, b=std, index=idx).numpy()
        assert np.array_equal(a.view(np.uint32), O.ref_normal(seed, 0x1D, idx, n, std).view(np.uint32))
        h = materialize(n, seed, b=std, index=idx, dtype=torch.bfloat16).float().numpy()
        assert np.array_equal(h.view(np.uint32), O.bf16_round(O.ref_normal(seed, 0x1D, idx, n, std))
                              .view(np.uint32))
    outs = materialize_parallel([1000, 3000], 4, torch.float32, scales=[1.0, 0.5])
    assert np.array_equal(outs[1].numpy(), O.ref_normal(4, 0x1D, 1, 3000, 0.5))
    c = materialize(10, 0, "const", 2.5).numpy()
    assert (c == 2.5).all()
    with pytest.raises(A.InvalidArgument, match="a <= b"):
        materialize(10, 0, "uniform", 1.0, 0.0)


def test_host_copy_concurrent_callers():
    """Several threads using the copy pool at once (the host jobs' issuer
    threads and other pipelines do): every batch completes, byte for byte."""
    import threading
    rng = np.random.default_rng(7)
    srcs = [rng.integers(0, 256, (3 << 20) + 17 * i, dtype=np.uint8) for i in range(6)]
    dsts = [np.zeros_like(s) for s in srcs]
    errs = []

    def run(i):
        for _ in range(5):
            if L.lib.agq_host_copy(dsts[i].ctypes.data, srcs[i].ctypes.data, srcs[i].nbytes) != 0:
                errs.append(i)

    ts = [threading.Thread(target=run, args=(i,)) for i in range(len(srcs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs
    for s, d in zip(srcs, dsts):
        assert np.array_equal(s, d)
