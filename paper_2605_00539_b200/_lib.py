"""ctypes binding of libagq_cuda.so (the C ABI in include/agq_cuda.h).

The product path has no CPU fallback: if the in-tree library is missing this
module raises at import time, and every device entry point returns
AGQ_ERR_CUDA without a B200.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("AGQ_LIB") or os.path.join(_HERE, "libagq_cuda.so")

AGQ_OK, AGQ_ERR_INVALID_ARGUMENT, AGQ_ERR_RUNTIME, AGQ_ERR_CUDA, AGQ_ERR_NCCL = range(5)
AGQ_F32, AGQ_BF16 = 0, 1
AGQ_CODES_PACKED, AGQ_CODES_BYTES = 0, 1
AGQ_OP_QUANTIZE, AGQ_OP_DEQUANTIZE, AGQ_OP_ACCUMULATE, AGQ_OP_ALLREDUCE = range(4)
AGQ_AR_NCCL, AGQ_AR_FUSED_P2P, AGQ_AR_PUSH_P2P, AGQ_AR_ONESHOT_P2P = 0, 1, 2, 3
AGQ_MAX_WORLD = 16
INT64_MAX = (1 << 63) - 1


class AgqErrors(C.Structure):
    """Mirror of agq_errors (device-resident error record)."""

    _fields_ = [
        ("nonfinite_block", C.c_longlong),
        ("bad_scale_block", C.c_longlong),
        ("bad_code_index", C.c_longlong),
        ("nonfinite_local", C.c_longlong),
        ("overflow_block", C.c_longlong),
        ("saturated", C.c_ulonglong),
    ]


class AgqTraceEvent(C.Structure):
    """Mirror of agq_trace_event (collective.hpp:50-57 TraceEvent)."""

    _fields_ = [("phase", C.c_int), ("sender", C.c_int), ("receiver", C.c_int),
                ("reserved", C.c_int), ("chunk_start", C.c_uint64), ("chunk_len", C.c_uint64),
                ("payload_bytes", C.c_uint64)]


class AgqSegment(C.Structure):
    _fields_ = [("x", C.c_void_p), ("codes", C.c_void_p), ("scales", C.c_void_p),
                ("n", C.c_uint64)]


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class ProtocolError(RuntimeError):
    """std::runtime_error in the reference."""


class CudaError(RuntimeError):
    pass


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the AGoQ hot path has no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, U64, I, U32, S = C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, C.c_void_p
    sig = {
        "agq_version": (C.c_char_p, []),
        "agq_last_error": (C.c_char_p, []),
        "agq_device_ok": (I, []),
        "agq_launch_count": (C.c_ulonglong, []),
        "agq_errors_reset": (I, [P, S]),
        "agq_errors_message": (I, [C.POINTER(AgqErrors), I, C.c_char_p, C.c_size_t]),
        "agq_num_blocks": (U64, [U64, U32]),
        "agq_packed_bytes": (U64, [U64, I]),
        "agq_check_codec_args": (I, [I, U32, I]),
        "agq_quantize": (I, [P, I, U64, I, U32, I, P, I, P, P, S]),
        "agq_dequantize": (I, [P, I, P, U64, I, U32, I, P, I, I, P, S]),
        "agq_quantize_grouped": (I, [C.POINTER(AgqSegment), I, I, I, I, P, S]),
        "agq_quantize_roundtrip": (I, [P, I, U64, I, U32, I, P, I, P, P, I, P, S]),
        "agq_roundtrip_host": (I, [P, U64, I, U32, I, P]),
        "agq_dequantize_grouped": (I, [C.POINTER(AgqSegment), I, I, I, I, I, P, S]),
        "agq_pack_codes": (I, [P, U64, I, P, S]),
        "agq_unpack_codes": (I, [P, U64, I, P, S]),
        "agq_fp8_accumulate": (I, [P, P, P, I, U64, U32, I, P, P, P, S]),
        "agq_fp8_reduce_requant": (I, [I, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), U64, U32,
                                       I, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), P, S]),
        "agq_chunk_assignment": (I, [U64, U32, I, C.POINTER(C.c_uint64)]),
        "agq_allreduce_simulated": (I, [I, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), U64, U32,
                                        P, P, P, S]),
        "agq_allreduce_naive_simulated": (I, [I, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), U64,
                                              U32, P, P, P, P, S]),
        "agq_comm_unique_id": (I, [C.c_char_p]),
        "agq_comm_init": (I, [C.POINTER(C.c_void_p), C.c_char_p, I, I, I]),
        "agq_comm_p2p_export": (I, [P, U64, C.c_char_p]),
        "agq_comm_p2p_open": (I, [P, C.c_char_p]),
        "agq_comm_p2p_buffers": (I, [P, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]),
        "agq_comm_destroy": (I, [P]),
        "agq_comm_rank": (I, [P]),
        "agq_comm_size": (I, [P]),
        "agq_comm_set_timeout": (I, [P, C.c_double]),
        "agq_comm_last_trace": (I, [P, C.POINTER(AgqTraceEvent), I, C.POINTER(C.c_int),
                                    C.POINTER(C.c_ulonglong)]),
        "agq_fill_input": (I, [C.c_uint64, C.c_uint64, C.c_uint64, I, C.c_double, C.c_double,
                               I, P, U64]),
        "agq_allreduce_fp8": (I, [P, P, P, U64, U32, I, P, S]),
        "agq_allreduce_naive_fp8": (I, [P, P, P, U64, U32, P, P, S]),
        "agq_allreduce_bf16_nccl": (I, [P, P, U64, S]),
        "agq_quantize_host": (I, [P, U64, I, U32, I, P, P]),
        "agq_host_pipeline_stats": (I, [C.POINTER(C.c_double), I]),
        "agq_host_copy": (I, [P, P, U64]),
        "agq_quantize_host_begin": (I, [P, U64, I, U32, I, P]),
        "agq_dequantize_host_begin": (I, [P, P, U64, I, U32, I, P]),
        "agq_roundtrip_host_begin": (I, [P, U64, I, U32, I, P]),
        "agq_local_accumulate_host_begin": (I, [P, P, U64, U32, P, I, P]),
        "agq_host_job_finish": (I, [P, P, P]),
        "agq_dequantize_host": (I, [P, P, U64, I, U32, I, P]),
        "agq_local_accumulate_host": (I, [P, P, U64, U32, P, I, P, P]),
        "agq_allreduce_simulated_host": (I, [I, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), U64,
                                             U32, I, P, P, C.POINTER(C.c_uint64),
                                             C.POINTER(C.c_uint64)]),
        "agq_stored_activation_counts": (I, [I, I, I, C.POINTER(C.c_int)]),
        "agq_plan_bit_widths": (I, [I, I, I, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                    C.POINTER(C.c_int)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

EXPORTED = (
    "agq_version agq_last_error agq_device_ok agq_launch_count agq_errors_reset "
    "agq_errors_message agq_num_blocks agq_packed_bytes agq_check_codec_args agq_quantize "
    "agq_dequantize agq_quantize_roundtrip agq_quantize_grouped agq_dequantize_grouped "
    "agq_pack_codes agq_unpack_codes agq_roundtrip_host "
    "agq_fp8_accumulate agq_fp8_reduce_requant agq_chunk_assignment agq_allreduce_simulated "
    "agq_allreduce_naive_simulated agq_comm_unique_id agq_comm_init agq_comm_p2p_export "
    "agq_comm_p2p_open agq_comm_p2p_buffers agq_comm_destroy agq_comm_rank agq_comm_size "
    "agq_comm_set_timeout agq_comm_last_trace agq_fill_input "
    "agq_allreduce_fp8 agq_allreduce_naive_fp8 agq_allreduce_bf16_nccl agq_quantize_host agq_dequantize_host "
    "agq_local_accumulate_host agq_host_pipeline_stats agq_host_copy agq_quantize_host_begin agq_dequantize_host_begin agq_roundtrip_host_begin agq_local_accumulate_host_begin agq_host_job_finish agq_allreduce_simulated_host agq_stored_activation_counts "
    "agq_plan_bit_widths").split()


def raise_status(st: int, msg: str | None = None) -> None:
    if st == AGQ_OK:
        return
    text = msg if msg is not None else (lib.agq_last_error() or b"").decode()
    if st == AGQ_ERR_INVALID_ARGUMENT:
        raise InvalidArgument(text)
    if st == AGQ_ERR_RUNTIME:
        raise ProtocolError(text)
    raise CudaError(text)


def check(st: int) -> None:
    raise_status(st)


def errors_message(h: AgqErrors, op: int) -> None:
    buf = C.create_string_buffer(256)
    st = lib.agq_errors_message(C.byref(h), op, buf, 256)
    raise_status(st, buf.value.decode())


def ptr_array(ptrs) -> "C.Array":
    arr = (C.c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
