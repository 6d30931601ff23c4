"""TEST INFRASTRUCTURE: ctypes access to the CPU oracle.

* `orc`  — oracle/liboracle.so, the plain-C restatement (always present once
  built; travels to the GPU box).
* `ref`  — oracle/_ref/libagq_ref.so, the reference headers compiled as-is
  (present where it was built; also travels). None if absent.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline use this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libagq_ref.so")

P = C.c_void_p
U8P = C.POINTER(C.c_uint8)
F32P = C.POINTER(C.c_float)


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)


def _load_orc():
    if not os.path.exists(ORACLE_SO):
        build_oracle()
    L = C.CDLL(ORACLE_SO)
    sz, I, U32 = C.c_size_t, C.c_int, C.c_uint32
    L.oracle_fp8_encode.restype = C.c_uint8
    L.oracle_fp8_encode.argtypes = [C.c_double, C.POINTER(C.c_int)]
    L.oracle_fp8_decode.restype = C.c_double
    L.oracle_fp8_decode.argtypes = [C.c_uint8]
    L.oracle_fp4_encode.restype = C.c_uint8
    L.oracle_fp4_encode.argtypes = [C.c_double]
    L.oracle_fp4_decode.restype = C.c_double
    L.oracle_fp4_decode.argtypes = [C.c_uint8]
    L.oracle_code_unit_value.restype = C.c_double
    L.oracle_code_unit_value.argtypes = [I, I, C.c_uint8]
    L.oracle_quantize.argtypes = [P, sz, I, U32, I, P, P, C.c_char_p, sz]
    L.oracle_dequantize.argtypes = [P, P, sz, I, U32, I, P, C.c_char_p, sz]
    L.oracle_pack_codes.restype = sz
    L.oracle_pack_codes.argtypes = [P, sz, I, P]
    L.oracle_unpack_codes.argtypes = [P, sz, I, sz, P]
    L.oracle_dump_size.restype = sz
    L.oracle_dump_size.argtypes = [sz, I, U32, I]
    L.oracle_dump.argtypes = [P, P, sz, I, U32, I, P, I, P]
    L.oracle_round_bf16.restype = C.c_float
    L.oracle_round_bf16.argtypes = [C.c_float]
    L.oracle_round_fp16.restype = C.c_float
    L.oracle_round_fp16.argtypes = [C.c_float]
    L.oracle_local_accumulate.argtypes = [P, P, sz, U32, P, I, P, P, C.c_char_p, sz]
    L.oracle_chunk_assignment.argtypes = [sz, U32, I, P]
    L.oracle_allreduce_oracle.argtypes = [I, sz, U32, P, P, P, C.c_char_p, sz]
    L.oracle_allreduce_decomposed.argtypes = [I, sz, U32, P, P, P, P, C.c_char_p, sz]
    L.oracle_allreduce_naive.argtypes = [I, sz, U32, P, P, P, P, C.POINTER(C.c_uint64),
                                         C.c_char_p, sz]
    L.oracle_stored_activation_counts.argtypes = [I, I, I, P]
    L.oracle_plan_bit_widths.argtypes = [I, I, I, P, P, P]
    L.oracle_plan_reuse.argtypes = [I, I, I, I, P, C.POINTER(C.c_double),
                                    C.POINTER(C.c_double), C.POINTER(C.c_int)]
    return L


def _load_ref():
    if not os.path.exists(REF_SO):
        return None
    L = C.CDLL(REF_SO)
    sz, I, U32 = C.c_size_t, C.c_int, C.c_uint32
    L.ref_fp8_encode.restype = C.c_uint8
    L.ref_fp8_encode.argtypes = [C.c_double, C.POINTER(C.c_int)]
    L.ref_fp8_decode.restype = C.c_double
    L.ref_fp8_decode.argtypes = [C.c_uint8]
    L.ref_fp4_encode.restype = C.c_uint8
    L.ref_fp4_encode.argtypes = [C.c_double]
    L.ref_fp4_decode.restype = C.c_double
    L.ref_fp4_decode.argtypes = [C.c_uint8]
    L.ref_round_bf16.restype = C.c_float
    L.ref_round_bf16.argtypes = [C.c_float]
    L.ref_round_fp16.restype = C.c_float
    L.ref_round_fp16.argtypes = [C.c_float]
    L.ref_fill_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_float, C.c_float, P, sz]
    L.ref_fill_normal_seed.argtypes = [C.c_uint64, C.c_float, P, sz]
    L.ref_quantize.argtypes = [P, sz, I, U32, I, P, P, C.c_char_p, sz]
    L.ref_dequantize.argtypes = [P, P, sz, I, U32, I, P, C.c_char_p, sz]
    L.ref_quantize_mt.argtypes = [P, sz, I, U32, I, P, P, I]
    L.ref_dequantize_mt.argtypes = [P, P, sz, I, U32, I, P, I]
    L.ref_pack_codes.restype = sz
    L.ref_pack_codes.argtypes = [P, sz, I, P]
    L.ref_dump_quantized.restype = C.c_longlong
    L.ref_dump_quantized.argtypes = [P, sz, I, U32, I, P, I, P, sz]
    L.ref_local_accumulate.argtypes = [P, P, sz, U32, P, I, P, P, C.c_char_p, sz]
    L.ref_local_accumulate_mt.argtypes = [P, P, sz, U32, P, I, P, P, I]
    L.ref_chunk_assignment.argtypes = [sz, U32, I, P, C.c_char_p, sz]
    L.ref_allreduce.argtypes = [I, I, sz, U32, P, P, P, P, P, C.POINTER(C.c_uint64), P, sz,
                                C.POINTER(C.c_size_t), C.POINTER(C.c_int), C.c_char_p, sz]
    L.ref_allreduce_oracle.argtypes = [I, sz, U32, P, P, P, C.c_char_p, sz]
    return L


orc = _load_orc()
ref = _load_ref()

LINEAR, FP4, FP8 = 0, 1, 2


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class OracleError(Exception):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


def _err():
    return C.create_string_buffer(256)


def quantize(x: np.ndarray, bits: int, block: int = 128, codec: int = LINEAR, lib=None):
    """(codes uint8 one per element, scales float32)."""
    L = lib or orc
    x = np.ascontiguousarray(x, dtype=np.float32)
    n = x.size
    nb = (n + block - 1) // block if block else 0
    codes = np.empty(n, np.uint8)
    scales = np.empty(nb, np.float32)
    e = _err()
    fn = L.oracle_quantize if L is orc else L.ref_quantize
    st = fn(_p(x), n, bits, block, codec, _p(codes), _p(scales), e, 256)
    if st:
        raise OracleError(st, e.value.decode())
    return codes, scales


def dequantize(codes, scales, bits, block=128, codec=LINEAR, lib=None):
    L = lib or orc
    codes = np.ascontiguousarray(codes, np.uint8)
    scales = np.ascontiguousarray(scales, np.float32)
    out = np.empty(codes.size, np.float32)
    e = _err()
    fn = L.oracle_dequantize if L is orc else L.ref_dequantize
    st = fn(_p(codes), _p(scales), codes.size, bits, block, codec, _p(out), e, 256)
    if st:
        raise OracleError(st, e.value.decode())
    return out


def pack(codes, bits, lib=None):
    L = lib or orc
    codes = np.ascontiguousarray(codes, np.uint8)
    out = np.empty((codes.size * bits + 7) // 8 + 1, np.uint8)
    fn = L.oracle_pack_codes if L is orc else L.ref_pack_codes
    k = fn(_p(codes), codes.size, bits, _p(out))
    return out[:k]


def unpack(packed, bits, count):
    packed = np.ascontiguousarray(packed, np.uint8)
    out = np.empty(count, np.uint8)
    st = orc.oracle_unpack_codes(_p(packed), packed.size, bits, count, _p(out))
    if st:
        raise OracleError(st, "tensor dump: packed codes truncated")
    return out


def local_accumulate(codes, scales, local, precision=0, block=128, lib=None):
    L = lib or orc
    codes = np.ascontiguousarray(codes, np.uint8)
    scales = np.ascontiguousarray(scales, np.float32)
    local = np.ascontiguousarray(local, np.float32)
    oc = np.empty_like(codes)
    os_ = np.empty_like(scales)
    e = _err()
    fn = L.oracle_local_accumulate if L is orc else L.ref_local_accumulate
    st = fn(_p(codes), _p(scales), codes.size, block, _p(local), precision, _p(oc), _p(os_), e,
            256)
    if st:
        raise OracleError(st, e.value.decode())
    return oc, os_


def _ptrs(arrs):
    a = (C.c_void_p * len(arrs))()
    for i, x in enumerate(arrs):
        a[i] = x.ctypes.data
    return a


def allreduce_decomposed(codes_list, scales_list, block=128):
    n = codes_list[0].size
    world = len(codes_list)
    codes_list = [np.ascontiguousarray(c, np.uint8) for c in codes_list]
    scales_list = [np.ascontiguousarray(s, np.float32) for s in scales_list]
    oc = np.empty(n, np.uint8)
    os_ = np.empty(scales_list[0].size, np.float32)
    e = _err()
    st = orc.oracle_allreduce_decomposed(world, n, block, _ptrs(codes_list), _ptrs(scales_list),
                                         _p(oc), _p(os_), e, 256)
    if st:
        raise OracleError(st, e.value.decode())
    return oc, os_


def allreduce_oracle(codes_list, scales_list, block=128):
    n = codes_list[0].size
    out = np.empty(n, np.float32)
    e = _err()
    codes_list = [np.ascontiguousarray(c, np.uint8) for c in codes_list]
    scales_list = [np.ascontiguousarray(s, np.float32) for s in scales_list]
    st = orc.oracle_allreduce_oracle(len(codes_list), n, block, _ptrs(codes_list),
                                     _ptrs(scales_list), _p(out), e, 256)
    if st:
        raise OracleError(st, e.value.decode())
    return out


def allreduce_naive(codes_list, scales_list, block=128):
    n = codes_list[0].size
    codes_list = [np.ascontiguousarray(c, np.uint8) for c in codes_list]
    scales_list = [np.ascontiguousarray(s, np.float32) for s in scales_list]
    oc = np.empty(n, np.uint8)
    os_ = np.empty(scales_list[0].size, np.float32)
    ov = C.c_uint64(0)
    e = _err()
    st = orc.oracle_allreduce_naive(len(codes_list), n, block, _ptrs(codes_list),
                                    _ptrs(scales_list), _p(oc), _p(os_), C.byref(ov), e, 256)
    if st:
        raise OracleError(st, e.value.decode())
    return oc, os_, int(ov.value)


def ref_allreduce(protocol, codes_list, scales_list, block=128, schedule=None):
    """The reference's own allreduce_decomposed (0) / allreduce_naive_fp8 (1)."""
    n = codes_list[0].size
    world = len(codes_list)
    codes_list = [np.ascontiguousarray(c, np.uint8) for c in codes_list]
    scales_list = [np.ascontiguousarray(s, np.float32) for s in scales_list]
    oc = np.empty(n, np.uint8)
    os_ = np.empty(scales_list[0].size, np.float32)
    ov = C.c_uint64(0)
    cap = 4 * world * world + 16
    trace = np.zeros(cap * 6, np.uint64)
    nev = C.c_size_t(0)
    same = C.c_int(0)
    sched = None
    if schedule is not None:
        sarr = (C.c_int * world)(*schedule)
        sched = C.cast(sarr, C.c_void_p)
    e = _err()
    st = ref.ref_allreduce(protocol, world, n, block, _ptrs(codes_list), _ptrs(scales_list), sched,
                           _p(oc), _p(os_), C.byref(ov), _p(trace), cap, C.byref(nev),
                           C.byref(same), e, 256)
    if st:
        raise OracleError(st, e.value.decode())
    ev = trace[: 6 * nev.value].reshape(-1, 6)
    return oc, os_, int(ov.value), ev, bool(same.value)


def ref_normal(root, stream, index, n, std=1.0, mean=0.0):
    out = np.empty(n, np.float32)
    ref.ref_fill_normal(root, stream, index, mean, std, _p(out), n)
    return out


def ref_normal_seed(seed, n, std=1.0):
    out = np.empty(n, np.float32)
    ref.ref_fill_normal_seed(seed, std, _p(out), n)
    return out


def bf16_round(x: np.ndarray) -> np.ndarray:
    """RNE to bf16 (values kept as float32), = round_bf16 of collective.hpp."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def fp8_decode_table() -> np.ndarray:
    return np.array([orc.oracle_fp8_decode(b) for b in range(256)], np.float64)
