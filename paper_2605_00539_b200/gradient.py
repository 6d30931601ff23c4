"""L2a gradient path on device tensors — mirror of collective.hpp:20-333,
338-431 (local_accumulate, ChunkAssignment, the decomposed all-reduce and the
naive FP8 ring), running the sm_100a kernels through the C ABI.

The reference simulates P workers inside one process (WorkerState); the
`*_simulated` functions keep that contract on ONE device (all workers' FP8
gradients resident in HBM). Real one-process-per-GPU ranks use
collective.Communicator.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib as L
from .codec import CodecKind, ErrorRecord, QuantizedTensor, _require_cuda, _stream, validate


class AccumulatePrecision(enum.IntEnum):  # collective.hpp:99
    Fp32 = 0
    Bf16 = 1
    Fp16 = 2


def _check_fp8(q: QuantizedTensor, what: str):
    if q.codec_kind != CodecKind.Fp8E4M3:
        raise L.InvalidArgument(what)
    if q.packed and q.bit_width != 8:
        raise L.InvalidArgument(what)


def local_accumulate(main: QuantizedTensor, local_grad: torch.Tensor,
                     precision: AccumulatePrecision = AccumulatePrecision.Fp32,
                     in_place: bool = False, stream=None, check: bool = True,
                     errors: ErrorRecord | None = None) -> QuantizedTensor:
    """collective.hpp:128-147: dequantize FP8 main, add local (optionally
    rounded to BF16/FP16), requantize with fresh block absmax scales."""
    _check_fp8(main, "main gradient must be FP8 E4M3")
    n = main.num_elements()
    if local_grad.numel() != n:
        raise L.InvalidArgument("local gradient shape mismatch")
    validate(main)  # dequantize_blockwise's structural checks (data checks on device)
    _require_cuda(local_grad, "local_grad")
    ldt = L.AGQ_BF16 if local_grad.dtype == torch.bfloat16 else L.AGQ_F32
    if local_grad.dtype not in (torch.float32, torch.bfloat16):
        raise L.InvalidArgument("local gradient must be float32 or bfloat16")
    if in_place:
        out = main
    else:
        out = QuantizedTensor(torch.empty_like(main.codes), torch.empty_like(main.scales), 8,
                              main.block_size, main.shape, CodecKind.Fp8E4M3, main.packed)
    err = errors if errors is not None else ErrorRecord(main.codes.device)
    err.reset(stream)
    L.check(L.lib.agq_fp8_accumulate(main.codes.data_ptr(), main.scales.data_ptr(),
                                     local_grad.data_ptr(), ldt, n, main.block_size,
                                     int(precision), out.codes.data_ptr(), out.scales.data_ptr(),
                                     err.ptr, _stream(stream)))
    if check:
        err.raise_if_any(L.AGQ_OP_ACCUMULATE)
    return out


@dataclass
class ChunkAssignment:  # collective.hpp:20-40
    ranges: list

    @staticmethod
    def block_aligned(n: int, block: int, workers: int) -> "ChunkAssignment":
        arr = (C.c_uint64 * (2 * max(workers, 1)))()
        L.check(L.lib.agq_chunk_assignment(n, block, workers, arr))
        return ChunkAssignment([(int(arr[2 * r]), int(arr[2 * r + 1])) for r in range(workers)])


def round_bf16(x: float) -> float:
    """collective.hpp:101-110 (host scalar)."""
    import struct
    u = struct.unpack("<I", struct.pack("<f", x))[0]
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return struct.unpack("<f", struct.pack("<I", u & 0xFFFFFFFF))[0]


def _check_world(mains: Sequence[QuantizedTensor]):
    if not mains:
        raise L.InvalidArgument("no workers")
    if len(mains) > L.AGQ_MAX_WORLD:
        raise L.InvalidArgument(f"at most {L.AGQ_MAX_WORLD} workers")
    for q in mains:
        _check_fp8(q, "worker gradients are FP8 E4M3 tensors")
    s0, b0 = mains[0].shape, mains[0].block_size
    for q in mains:
        if q.shape != s0 or q.block_size != b0:
            raise L.InvalidArgument("all-reduce aborted: main gradient shapes must match")
        validate(q)  # collective.hpp:166 (structural part; data checks on device)


def allreduce_simulated(mains: Sequence[QuantizedTensor], stream=None, check: bool = True,
                        errors: ErrorRecord | None = None,
                        out: QuantizedTensor | None = None) -> QuantizedTensor:
    """allreduce_decomposed (collective.hpp:226-333) for in-process workers on
    one device: the tensor every worker holds afterwards."""
    _check_world(mains)
    n, blk = mains[0].num_elements(), mains[0].block_size
    if out is None:
        out = QuantizedTensor(torch.empty_like(mains[0].codes), torch.empty_like(mains[0].scales),
                              8, blk, mains[0].shape, CodecKind.Fp8E4M3, mains[0].packed)
    err = errors if errors is not None else ErrorRecord(mains[0].codes.device)
    err.reset(stream)
    pc = L.ptr_array([q.codes.data_ptr() for q in mains])
    ps = L.ptr_array([q.scales.data_ptr() for q in mains])
    L.check(L.lib.agq_allreduce_simulated(len(mains), pc, ps, n, blk, out.codes.data_ptr(),
                                          out.scales.data_ptr(), err.ptr, _stream(stream)))
    if check:
        err.raise_if_any(L.AGQ_OP_ALLREDUCE)
    return out


def allreduce_naive_simulated(mains: Sequence[QuantizedTensor], stream=None, events: bool = False):
    """allreduce_naive_fp8 (collective.hpp:338-431): returns (tensor,
    overflow_elements[, per-worker overflow_events])."""
    _check_world(mains)
    n, blk = mains[0].num_elements(), mains[0].block_size
    out = QuantizedTensor(torch.empty_like(mains[0].codes), torch.empty_like(mains[0].scales), 8,
                          blk, mains[0].shape, CodecKind.Fp8E4M3, mains[0].packed)
    err = ErrorRecord(mains[0].codes.device).reset(stream)
    ev = torch.zeros(len(mains), dtype=torch.int64, device=mains[0].codes.device)
    pc = L.ptr_array([q.codes.data_ptr() for q in mains])
    ps = L.ptr_array([q.scales.data_ptr() for q in mains])
    L.check(L.lib.agq_allreduce_naive_simulated(len(mains), pc, ps, n, blk, out.codes.data_ptr(),
                                                out.scales.data_ptr(), err.ptr, ev.data_ptr(),
                                                _stream(stream)))
    h = err.raise_if_any(L.AGQ_OP_ALLREDUCE)
    if events:
        return out, int(h.saturated), [int(v) for v in ev.cpu().tolist()]
    return out, int(h.saturated)


@dataclass
class TraceEvent:  # collective.hpp:50-57
    phase: str
    sender: int
    receiver: int
    chunk_start: int
    chunk_len: int
    payload_bytes: int


def decomposed_trace(n: int, block: int, world: int) -> list:
    """The MessageTrace allreduce_decomposed records (collective.hpp:239-300):
    the message schedule is a pure function of (n, block, world)."""
    a = ChunkAssignment.block_aligned(n, block, world).ranges
    ev = []
    for s in range(world):
        for r in range(world):
            b, e = a[r]
            if r == s or b == e:
                continue
            nsc = (e + block - 1) // block - b // block
            ev.append(TraceEvent("all_to_all", s, r, b, e - b, (e - b) + 4 * nsc))
    for s in range(world):
        b, e = a[s]
        if b == e:
            continue
        nsc = (e - b + block - 1) // block
        for r in range(world):
            if r != s:
                ev.append(TraceEvent("all_gather", s, r, b, e - b, (e - b) + 4 * nsc))
    return ev


def naive_trace(n: int, block: int, world: int) -> list:
    """The MessageTrace allreduce_naive_fp8 records (collective.hpp:356-421):
    P-1 ring steps in which rank r sends chunk (r - step) mod P to r+1, then
    the all-gather of chunk c from its owner (c - 1) mod P to every other rank."""
    a = ChunkAssignment.block_aligned(n, block, world).ranges

    def payload(b, e):
        return (e - b) + 4 * ((e + block - 1) // block - b // block)

    ev = []
    for step in range(world - 1):
        for r in range(world):
            b, e = a[(r - step) % world]
            if b != e:
                ev.append(TraceEvent("reduce_scatter", r, (r + 1) % world, b, e - b, payload(b, e)))
    for c in range(world):
        owner = 0 if world == 1 else (c - 1) % world
        b, e = a[c]
        if b == e:
            continue
        for r in range(world):
            if r != owner:
                ev.append(TraceEvent("all_gather", owner, r, b, e - b, payload(b, e)))
    return ev
