"""Decomposed 8-bit all-reduce across real ranks (one process per GPU).

Replaces allreduce_decomposed (collective.hpp:226-333) when the workers are
GPUs of one NVLink/NVSwitch box. torch.distributed is only the plumbing that
carries the NCCL unique id and the CUDA IPC handles between processes; the
data path is libagq_cuda.so (NCCL grouped send/recv + the reduce-requant
kernel, or the fused NVLink peer-memory kernel).
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L
from .codec import CodecKind, ErrorRecord, QuantizedTensor, _stream, validate
from .gradient import TraceEvent

PHASES = ("all_to_all", "all_gather")


class _CudaArray:
    """Zero-copy view of raw device memory for torch.as_tensor."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class Communicator:
    ALGOS = {"nccl": L.AGQ_AR_NCCL, "p2p": L.AGQ_AR_FUSED_P2P, "push": L.AGQ_AR_PUSH_P2P,
             "oneshot": L.AGQ_AR_ONESHOT_P2P}
    ONESHOT_MAX = 1 << 20  # elements: the one-shot inbox (csrc/collective.cu)
    # auto picks the one-shot algorithm while n * (P - 1) stays below this:
    # it sends 2 (P - 1) x the decomposed protocol's bytes but skips its
    # second exchange and both barriers (profiles/r02_oneshot_*.log)
    ONESHOT_AUTO = 3 << 19

    def __init__(self, group=None, device: int | None = None, p2p_capacity: int = 0,
                 timeout_s: float | None = None, nccl: bool = True):
        """nccl=False: a P2P-only communicator (the NVLink algorithms only, no
        NCCL communicator); several ranks may then share one GPU."""
        import torch.distributed as dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = torch.cuda.current_device() if device is None else device
        self.nccl = nccl
        uid = None
        if nccl:
            uid = C.create_string_buffer(128)
            if self.rank == 0:
                L.check(L.lib.agq_comm_unique_id(uid))
            t = torch.frombuffer(bytearray(uid.raw), dtype=torch.uint8).clone()
            t = self._bcast_bytes(t, group)
            uid = C.create_string_buffer(bytes(t.tolist()), 128)
        self._h = C.c_void_p()
        L.check(L.lib.agq_comm_init(C.byref(self._h), uid, self.world, self.rank, self.device))
        self._group = group
        self.p2p_capacity = 0
        if timeout_s is not None:
            self.set_timeout(timeout_s)
        if p2p_capacity:
            self.enable_p2p(p2p_capacity)

    @staticmethod
    def _bcast_bytes(t: torch.Tensor, group):
        import torch.distributed as dist
        if dist.get_backend(group) == "nccl":
            d = t.cuda()
            dist.broadcast(d, 0, group=group)
            return d.cpu()
        dist.broadcast(t, 0, group=group)
        return t

    def enable_p2p(self, capacity: int):
        """Allocate + IPC-export this rank's symmetric FP8 buffer, open all
        peers' (collective over the group)."""
        import torch.distributed as dist
        h = C.create_string_buffer(256)
        L.check(L.lib.agq_comm_p2p_export(self._h, int(capacity), h))
        mine = torch.frombuffer(bytearray(h.raw), dtype=torch.uint8).clone()
        if dist.get_backend(self._group) == "nccl":
            outs = [torch.empty(256, dtype=torch.uint8, device="cuda") for _ in range(self.world)]
            dist.all_gather(outs, mine.cuda(), group=self._group)
            outs = [o.cpu() for o in outs]
        else:
            outs = [torch.empty(256, dtype=torch.uint8) for _ in range(self.world)]
            dist.all_gather(outs, mine, group=self._group)
        blob = b"".join(bytes(o.tolist()) for o in outs)
        L.check(L.lib.agq_comm_p2p_open(self._h, C.create_string_buffer(blob, len(blob))))
        self.p2p_capacity = int(capacity)

    def p2p_buffers(self, n: int):
        """(codes, scales) torch views of this rank's symmetric buffer for an
        n-element gradient; all-reducing these runs fully in place."""
        c, s = C.c_void_p(), C.c_void_p()
        L.check(L.lib.agq_comm_p2p_buffers(self._h, C.byref(c), C.byref(s)))
        nb = (n + 127) // 128
        codes = torch.as_tensor(_CudaArray(c.value, n, "|u1"), device=f"cuda:{self.device}")
        scales = torch.as_tensor(_CudaArray(s.value, nb, "<f4"), device=f"cuda:{self.device}")
        return codes, scales

    def set_timeout(self, seconds: float):
        """Device barrier timeout of the P2P algorithms (default 300 s). A
        timeout aborts the call on every rank ("peer did not arrive") and
        leaves the communicator failed: re-create it."""
        L.check(L.lib.agq_comm_set_timeout(self._h, float(seconds)))

    def _auto_algo(self, q: QuantizedTensor) -> str:
        # Depends only on state every rank shares (the collective
        # enable_p2p capacity, and n / block, equal on all ranks), never on
        # where this rank's tensor lives, so all ranks pick the same algorithm.
        n = q.num_elements()
        if self.p2p_capacity and n <= self.p2p_capacity and q.block_size == 128:
            if (n <= self.ONESHOT_MAX and self.world <= 8 and
                    n * (self.world - 1) <= self.ONESHOT_AUTO):
                return "oneshot"
            return "p2p"
        if not self.nccl:
            raise L.InvalidArgument("P2P-only communicator: enable_p2p with enough capacity")
        return "nccl"

    def allreduce_fp8(self, q: QuantizedTensor, algo: str = "auto", stream=None,
                      check: bool = True, errors: ErrorRecord | None = None) -> QuantizedTensor:
        """In place on this rank's FP8 gradient (one byte per code).

        algo: "nccl" (grouped send/recv + reduce kernel), "p2p" (one fused
        NVLink kernel), "push" (store-only NVLink variant), or "auto": the
        fused kernel whenever peer buffers are enabled and large enough
        (a tensor outside p2p_buffers is copied in and out), otherwise NCCL —
        all bit-identical. validate() runs first (collective.hpp:166)."""
        if q.codec_kind != CodecKind.Fp8E4M3:
            raise L.InvalidArgument("worker gradients are FP8 E4M3 tensors")
        if q.packed and q.bit_width != 8:
            raise L.InvalidArgument("worker gradients are FP8 E4M3 tensors")
        validate(q)
        if algo == "auto":
            algo = self._auto_algo(q)
        err = errors if errors is not None else ErrorRecord(q.codes.device)
        err.reset(stream)
        L.check(L.lib.agq_allreduce_fp8(self._h, q.codes.data_ptr(), q.scales.data_ptr(),
                                        q.num_elements(), q.block_size, self.ALGOS[algo], err.ptr,
                                        _stream(stream)))
        if check:
            err.raise_if_any(L.AGQ_OP_ALLREDUCE)
        return q

    def last_trace(self):
        """(events, moved): the messages this rank took part in during its
        last allreduce_fp8 (TraceEvent list, collective.hpp:50-57) as issued
        by the transfer code, and for the P2P algorithms the kernel's own
        counters of the phase-1 traffic (elements, block scales)."""
        cnt = C.c_int()
        moved = (C.c_ulonglong * 2)()
        L.check(L.lib.agq_comm_last_trace(self._h, None, 0, C.byref(cnt), moved))
        arr = (L.AgqTraceEvent * max(cnt.value, 1))()
        L.check(L.lib.agq_comm_last_trace(self._h, arr, cnt.value, C.byref(cnt), moved))
        ev = [TraceEvent(PHASES[e.phase], e.sender, e.receiver, e.chunk_start, e.chunk_len,
                         e.payload_bytes) for e in arr[:cnt.value]]
        return ev, (int(moved[0]), int(moved[1]))

    def gather_trace(self):
        """The reference's MessageTrace of the last all-reduce across ALL
        ranks: the union of every rank's last_trace(), de-duplicated and in
        the reference's order (phase, then sender, then receiver;
        collective.hpp:239-248, :287-300)."""
        import torch.distributed as dist
        mine, _ = self.last_trace()
        allv = [None] * self.world
        dist.all_gather_object(allv, [tuple(e.__dict__.values()) for e in mine], group=self._group)
        uniq = {}
        for rank_events in allv:
            for t in rank_events:
                uniq[(PHASES.index(t[0]), t[1], t[2])] = TraceEvent(*t)
        return [uniq[k] for k in sorted(uniq)]

    def allreduce_naive_fp8(self, q: QuantizedTensor, stream=None):
        """allreduce_naive_fp8 (collective.hpp:338-431) across the ranks, in
        place: the overflow-prone FP8 ring strawman. Returns (q,
        overflow_elements, this rank's overflow_events) like the reference's
        CollectiveResult (events of the other ranks stay on those ranks)."""
        if q.codec_kind != CodecKind.Fp8E4M3:
            raise L.InvalidArgument("worker gradients are FP8 E4M3 tensors")
        if q.packed:
            raise L.InvalidArgument("the all-reduce takes one byte per code (packed=False)")
        err = ErrorRecord(q.codes.device).reset(stream)
        ev = torch.zeros(1, dtype=torch.int64, device=q.codes.device)
        L.check(L.lib.agq_allreduce_naive_fp8(self._h, q.codes.data_ptr(), q.scales.data_ptr(),
                                              q.num_elements(), q.block_size, err.ptr,
                                              ev.data_ptr(), _stream(stream)))
        h = err.raise_if_any(L.AGQ_OP_ALLREDUCE)
        return q, int(h.saturated), int(ev.item())

    def allreduce_bf16(self, t: torch.Tensor, stream=None) -> torch.Tensor:
        """Baseline: ncclAllReduce(bf16, sum) in place."""
        if t.dtype != torch.bfloat16:
            raise L.InvalidArgument("baseline expects bfloat16")
        L.check(L.lib.agq_allreduce_bf16_nccl(self._h, t.data_ptr(), t.numel(), _stream(stream)))
        return t

    def close(self):
        if self._h:
            L.lib.agq_comm_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
