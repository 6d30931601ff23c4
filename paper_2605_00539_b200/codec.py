"""L1 block codec on device tensors — Python mirror of the reference API in
/root/reference/proj/include/agq/quantize.hpp and tensor_io.hpp, running the
sm_100a kernels of libagq_cuda.so through the C ABI.

`quantize_blockwise` / `dequantize_blockwise` keep the reference's names,
argument meaning and exceptions (InvalidArgument == std::invalid_argument);
tensors live in HBM. Codes are stored packed (LSB-first bitstream at
`bit_width` bits, tensor_io.hpp:63-80) unless `packed=False` asks for the
reference's one-byte-per-element layout.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Sequence

import torch

from . import _lib as L


class CodecKind(enum.IntEnum):  # quantize.hpp:15-19
    SymmetricLinear = 0
    Fp4E2M1 = 1
    Fp8E4M3 = 2


kDefaultBlockSize = 128


@dataclass
class QuantizedTensor:  # quantize.hpp:40-50, device resident
    codes: torch.Tensor
    scales: torch.Tensor
    bit_width: int
    block_size: int = kDefaultBlockSize
    shape: tuple = ()
    codec_kind: CodecKind = CodecKind.SymmetricLinear
    packed: bool = True

    def num_elements(self) -> int:
        n = 1
        for d in self.shape:
            n *= int(d)
        return n

    def num_blocks(self) -> int:
        return int(self.scales.numel())

    def nbytes(self) -> int:
        return self.codes.numel() + 4 * self.scales.numel()


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class ErrorRecord:
    """Device-resident agq_errors record; `raise_if_any` syncs the stream.

    A record read back clean needs no reset before its next use: reset()
    then skips the reset kernel (the common path of every checked call).
    Handing out `ptr` (to a kernel) makes its state unknown again."""

    def __init__(self, device):
        self.t = torch.empty(C.sizeof(L.AgqErrors), dtype=torch.uint8, device=device)
        self._clean = False

    @property
    def ptr(self) -> int:
        self._clean = False
        return self.t.data_ptr()

    def reset(self, stream=None):
        if not self._clean:
            L.check(L.lib.agq_errors_reset(self.t.data_ptr(), _stream(stream)))
        return self

    def read(self) -> L.AgqErrors:
        raw = bytes(self.t.cpu().numpy().tobytes())
        h = L.AgqErrors.from_buffer_copy(raw)
        self._clean = raw == _CLEAN_RECORD
        return h

    def raise_if_any(self, op: int) -> L.AgqErrors:
        h = self.read()
        L.errors_message(h, op)
        return h


def _clean_record() -> bytes:
    """The bytes agq_errors_reset writes (index fields at INT64_MAX, counters 0)."""
    h = L.AgqErrors()
    for name, ctype in L.AgqErrors._fields_:
        setattr(h, name, 0 if ctype == C.c_ulonglong else (1 << 63) - 1)
    return bytes(h)


_CLEAN_RECORD = _clean_record()


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return L.AGQ_BF16
    if t.dtype == torch.float32:
        return L.AGQ_F32
    raise L.InvalidArgument(f"unsupported input dtype {t.dtype} (float32 or bfloat16)")


def _require_cuda(t: torch.Tensor, what: str):
    if not t.is_cuda:
        raise L.InvalidArgument(f"{what} must be a CUDA tensor (no CPU path)")
    if not t.is_contiguous():
        raise L.InvalidArgument(f"{what} must be contiguous")


def check_codec_args(bit_width: int, block_size: int, kind: CodecKind) -> None:
    """quantize.hpp:64-74; valid arguments return without a library call,
    invalid ones raise the library's (the reference's) message."""
    b, k = int(bit_width), int(kind)
    if 4 <= b <= 8 and int(block_size) >= 1 and (k == 0 or (k == 1 and b == 4) or (k == 2 and b == 8)):
        return
    L.check(L.lib.agq_check_codec_args(b, int(block_size), k))


def quantize_blockwise(x: torch.Tensor, bit_width: int, block_size: int = kDefaultBlockSize,
                       kind: CodecKind = CodecKind.SymmetricLinear, shape: Sequence[int] = (),
                       packed: bool = True, stream=None, check: bool = True,
                       errors: ErrorRecord | None = None) -> QuantizedTensor:
    """quantize.hpp:78-138 (+ pack_codes when packed). x: float32/bfloat16 CUDA."""
    check_codec_args(bit_width, block_size, kind)
    _require_cuda(x, "x")
    shape = tuple(int(d) for d in shape) if shape else (int(x.numel()),)
    n = 1
    for d in shape:
        n *= d
    if n != x.numel():
        raise L.InvalidArgument("shape does not match element count")
    nb = -(-n // block_size)  # agq_num_blocks
    ncode = -(-n * bit_width // 8) if packed else n  # agq_packed_bytes
    codes = torch.empty(ncode, dtype=torch.uint8, device=x.device)
    scales = torch.empty(nb, dtype=torch.float32, device=x.device)
    err = errors if errors is not None else (ErrorRecord(x.device) if check else None)
    s = _stream(stream)
    if err is not None:
        err.reset(stream)
    L.check(L.lib.agq_quantize(x.data_ptr(), _dtype_code(x), n, bit_width, block_size, int(kind),
                               codes.data_ptr(), L.AGQ_CODES_PACKED if packed else L.AGQ_CODES_BYTES,
                               scales.data_ptr(), err.ptr if err is not None else None, s))
    if check and err is not None:
        err.raise_if_any(L.AGQ_OP_QUANTIZE)
    return QuantizedTensor(codes, scales, bit_width, block_size, shape, CodecKind(kind), packed)


def validate(q: QuantizedTensor) -> None:
    """quantize.hpp:157-176 (argument/shape part; data checks run on device)."""
    check_codec_args(q.bit_width, q.block_size, q.codec_kind)
    n = q.num_elements()
    if q.scales.numel() != -(-n // q.block_size):  # agq_num_blocks
        raise L.InvalidArgument("quantized tensor: wrong number of scales")
    expect = -(-n * q.bit_width // 8) if q.packed else n  # agq_packed_bytes
    if q.codes.numel() != expect:
        raise L.InvalidArgument("quantized tensor: shape/code count mismatch")


_validate = validate  # (dequantize_grouped's `validate` flag shadows the name)


def dequantize_blockwise(q: QuantizedTensor, out_dtype: torch.dtype = torch.float32,
                         stream=None, check: bool = True, out: torch.Tensor | None = None,
                         errors: ErrorRecord | None = None) -> torch.Tensor:
    """quantize.hpp:178-189. float32 output is bit-identical to the reference;
    bfloat16 output is its round-to-nearest-even."""
    validate(q)
    n = q.num_elements()
    if out is None:
        out = torch.empty(n, dtype=out_dtype, device=q.codes.device)
    err = errors if errors is not None else (ErrorRecord(q.codes.device) if check else None)
    s = _stream(stream)
    if err is not None:
        err.reset(stream)
    L.check(L.lib.agq_dequantize(q.codes.data_ptr(),
                                 L.AGQ_CODES_PACKED if q.packed else L.AGQ_CODES_BYTES,
                                 q.scales.data_ptr(), n, q.bit_width, q.block_size,
                                 int(q.codec_kind), out.data_ptr(), _dtype_code(out),
                                 1 if err is not None else 0,
                                 err.ptr if err is not None else None, s))
    if check and err is not None:
        err.raise_if_any(L.AGQ_OP_DEQUANTIZE)
    return out.view(q.shape) if len(q.shape) > 1 else out


def code_unit_value(kind: CodecKind, bit_width: int, code: int) -> float:
    """quantize.hpp:142-155 (host scalar)."""
    if kind == CodecKind.SymmetricLinear:
        lv = (1 << (bit_width - 1)) - 1
        return (int(code) - lv) / lv
    if kind == CodecKind.Fp4E2M1:
        mag = (0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0)[code & 7]
        return (-mag if code & 8 else mag) / 6.0
    from .scalar import fp8_decode
    return fp8_decode(code) / 448.0


def pack_codes(codes: torch.Tensor, bit_width: int, stream=None) -> torch.Tensor:
    """tensor_io.hpp:63-80 on device."""
    _require_cuda(codes, "codes")
    n = codes.numel()
    out = torch.empty(int(L.lib.agq_packed_bytes(n, bit_width)), dtype=torch.uint8,
                      device=codes.device)
    L.check(L.lib.agq_pack_codes(codes.data_ptr(), n, bit_width, out.data_ptr(), _stream(stream)))
    return out


def unpack_codes(packed: torch.Tensor, bit_width: int, count: int, stream=None) -> torch.Tensor:
    """tensor_io.hpp:82-100 on device."""
    _require_cuda(packed, "packed")
    if packed.numel() < int(L.lib.agq_packed_bytes(count, bit_width)):
        raise L.ProtocolError("tensor dump: packed codes truncated")
    out = torch.empty(count, dtype=torch.uint8, device=packed.device)
    L.check(L.lib.agq_unpack_codes(packed.data_ptr(), count, bit_width, out.data_ptr(),
                                   _stream(stream)))
    return out


def _raise_grouped(err: "ErrorRecord", op: int, ns: Sequence[int]) -> None:
    """Raise the reference's exception for the first failing tensor of a
    grouped call. The device record holds group-global indices (blocks, and
    elements in block-padded coordinates); the reference processes the
    tensors one after the other, so the tensor with the lowest index fails
    first, with its own check order (code range before scales) and its own
    local index in the message. The exception carries `.segment`."""
    h = err.read()
    base = [0]
    for n in ns:
        base.append(base[-1] + (int(n) + 127) // 128)

    def seg_of(blk: int) -> int:
        for j in range(len(ns)):
            if blk < base[j + 1]:
                return j
        return len(ns) - 1

    fields = {"nonfinite_block": 1, "bad_code_index": 128, "bad_scale_block": 1}
    hits = []
    order = ["bad_code_index", "bad_scale_block"] if op == L.AGQ_OP_DEQUANTIZE else ["nonfinite_block"]
    for rank, name in enumerate(order):
        v = getattr(h, name)
        if v != L.INT64_MAX:
            hits.append((seg_of(v // fields[name]), rank, name, v))
    if not hits:
        return
    j, _, name, v = min(hits)
    loc = L.AgqErrors(L.INT64_MAX, L.INT64_MAX, L.INT64_MAX, L.INT64_MAX, L.INT64_MAX, 0)
    setattr(loc, name, v - base[j] * fields[name])
    try:
        L.errors_message(loc, op)
    except (L.InvalidArgument, L.ProtocolError) as e:
        e.segment = j
        raise


def quantize_grouped(xs: Sequence[torch.Tensor], bit_width: int,
                     kind: CodecKind = CodecKind.SymmetricLinear, stream=None,
                     check: bool = True, errors: ErrorRecord | None = None,
                     outs: Sequence[QuantizedTensor] | None = None) -> list[QuantizedTensor]:
    """One launch per 8 tensors over all tensors a pipeline stage stores
    (layers.hpp:266-301 for every layer of the stage, dbca.hpp:172-177 width;
    block 128, packed)."""
    if not xs:
        return []
    check_codec_args(bit_width, 128, kind)
    dt = _dtype_code(xs[0])
    qs = list(outs) if outs is not None else []
    segs = (L.AgqSegment * len(xs))()
    for i, x in enumerate(xs):
        _require_cuda(x, "x")
        if _dtype_code(x) != dt:
            raise L.InvalidArgument("grouped tensors must share a dtype")
        n = x.numel()
        if outs is None:
            q = QuantizedTensor(
                torch.empty(int(L.lib.agq_packed_bytes(n, bit_width)), dtype=torch.uint8,
                            device=x.device),
                torch.empty(int(L.lib.agq_num_blocks(n, 128)), dtype=torch.float32, device=x.device),
                bit_width, 128, tuple(x.shape), CodecKind(kind), True)
            qs.append(q)
        q = qs[i]
        segs[i] = L.AgqSegment(x.data_ptr(), q.codes.data_ptr(), q.scales.data_ptr(), n)
    err = errors if errors is not None else (ErrorRecord(xs[0].device) if check else None)
    if err is not None:
        err.reset(stream)
    L.check(L.lib.agq_quantize_grouped(segs, len(xs), dt, bit_width, int(kind),
                                       err.ptr if err is not None else None, _stream(stream)))
    if check and err is not None:
        _raise_grouped(err, L.AGQ_OP_QUANTIZE, [x.numel() for x in xs])
    return qs


def dequantize_grouped(qs: Sequence[QuantizedTensor], out_dtype: torch.dtype = torch.bfloat16,
                       stream=None, outs: Sequence[torch.Tensor] | None = None,
                       check: bool = True, errors: ErrorRecord | None = None,
                       validate: bool = True) -> list[torch.Tensor]:
    """dequantize_blockwise (quantize.hpp:178-189, validate :157-176 first)
    over a group of packed block-128 tensors in one launch per 8 tensors.
    With validate the device checks code range and scales of every tensor;
    `check` reads the record and raises the reference's exception."""
    if not qs:
        return []
    res = list(outs) if outs is not None else [
        torch.empty(q.shape, dtype=out_dtype, device=q.codes.device) for q in qs]
    segs = (L.AgqSegment * len(qs))()
    for i, q in enumerate(qs):
        if q.bit_width != qs[0].bit_width or q.codec_kind != qs[0].codec_kind or not q.packed:
            raise L.InvalidArgument("grouped tensors must share bits/codec and be packed")
        if q.block_size != 128:
            raise L.InvalidArgument("grouped tensors use block 128")
        _validate(q)
        segs[i] = L.AgqSegment(res[i].data_ptr(), q.codes.data_ptr(), q.scales.data_ptr(),
                               q.num_elements())
    err = errors if errors is not None else (
        ErrorRecord(qs[0].codes.device) if (validate or check) else None)
    if err is not None:
        err.reset(stream)
    L.check(L.lib.agq_dequantize_grouped(segs, len(qs), _dtype_code(res[0]), qs[0].bit_width,
                                         int(qs[0].codec_kind), 1 if validate else 0,
                                         err.ptr if err is not None else None, _stream(stream)))
    if check and validate and err is not None:
        _raise_grouped(err, L.AGQ_OP_DEQUANTIZE, [q.num_elements() for q in qs])
    return res


def quantize_roundtrip(x: torch.Tensor, bit_width: int, block_size: int = kDefaultBlockSize,
                       kind: CodecKind = CodecKind.SymmetricLinear, out_dtype=None, stream=None,
                       check: bool = True, errors: ErrorRecord | None = None):
    """quantize_blockwise + dequantize_blockwise of its result in one call
    (the round trip of quantize.hpp:193-196): (QuantizedTensor, reconstruction).
    SymmetricLinear BF16 in/out at block 128 is one fused kernel pass (x read
    once); bit-identical to the two calls."""
    check_codec_args(bit_width, block_size, kind)
    _require_cuda(x, "x")
    n = x.numel()
    out_dtype = out_dtype or x.dtype
    codes = torch.empty(int(L.lib.agq_packed_bytes(n, bit_width)), dtype=torch.uint8, device=x.device)
    scales = torch.empty(int(L.lib.agq_num_blocks(n, block_size)), dtype=torch.float32,
                         device=x.device)
    y = torch.empty(x.shape, dtype=out_dtype, device=x.device)
    err = errors if errors is not None else (ErrorRecord(x.device) if check else None)
    if err is not None:
        err.reset(stream)
    L.check(L.lib.agq_quantize_roundtrip(x.data_ptr(), _dtype_code(x), n, bit_width, block_size,
                                         int(kind), codes.data_ptr(), L.AGQ_CODES_PACKED,
                                         scales.data_ptr(), y.data_ptr(), _dtype_code(y),
                                         err.ptr if err is not None else None, _stream(stream)))
    if check and err is not None:
        err.raise_if_any(L.AGQ_OP_QUANTIZE)
    q = QuantizedTensor(codes, scales, bit_width, block_size, (n,), CodecKind(kind), True)
    return q, y


def roundtrip_relative_delta(x: torch.Tensor, bit_width: int, block_size: int = kDefaultBlockSize,
                             kind: CodecKind = CodecKind.SymmetricLinear) -> torch.Tensor:
    """quantize.hpp:193-206: x_hat = x (1 + delta); zero elements get 0."""
    _, y = quantize_roundtrip(x, bit_width, block_size, kind, out_dtype=torch.float32)
    back = y.reshape(-1).double()
    xd = x.reshape(-1).double()
    delta = torch.where(xd == 0, torch.zeros_like(xd), (back - xd) / xd)
    return delta
