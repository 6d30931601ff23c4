"""AGQT dump/load of device-resident quantized tensors (tensor_io.hpp:16-161).

The on-disk layout is header + FP32 scales + LSB-first packed codes. The GPU
codec already keeps codes in exactly that packed layout in HBM, so a dump is
two D2H copies (scales, codes) behind a 14 + 8*ndim byte header; a load is
two H2D copies. One-byte-per-element tensors are packed on the device first.
"""
from __future__ import annotations

import struct

import torch

from . import _lib as L
from .codec import CodecKind, QuantizedTensor, check_codec_args, pack_codes, unpack_codes

MAGIC = b"AGQT"
VERSION = 1


def dump_tensor(q: QuantizedTensor) -> bytes:
    check_codec_args(q.bit_width, q.block_size, q.codec_kind)
    n = q.num_elements()
    packed = q.codes if q.packed else pack_codes(q.codes, q.bit_width)
    if packed.numel() != int(L.lib.agq_packed_bytes(n, q.bit_width)):
        raise L.InvalidArgument("quantized tensor: shape/code count mismatch")
    head = MAGIC + struct.pack("<HBBIB", VERSION, int(q.codec_kind), q.bit_width, q.block_size,
                               len(q.shape))
    head += b"".join(struct.pack("<Q", int(d)) for d in q.shape)
    return head + q.scales.cpu().numpy().tobytes() + packed.cpu().numpy().tobytes()


def load_tensor(data: bytes, device="cuda", packed: bool = True) -> QuantizedTensor:
    if len(data) < 4 or data[:4] != MAGIC:
        raise L.ProtocolError("tensor dump: bad magic")
    if len(data) < 13:
        raise L.ProtocolError("tensor dump: truncated input")
    version, codec, bits, block, ndim = struct.unpack_from("<HBBIB", data, 4)
    if version != VERSION:
        raise L.ProtocolError(f"tensor dump: unsupported version {version}")
    if codec > 2:
        raise L.ProtocolError("tensor dump: unknown codec kind")
    off = 13
    if len(data) < off + 8 * ndim:
        raise L.ProtocolError("tensor dump: truncated input")
    shape = struct.unpack_from("<" + "Q" * ndim, data, off)
    off += 8 * ndim
    check_codec_args(bits, block, CodecKind(codec))
    n = 1
    for d in shape:
        n *= d
    nb = int(L.lib.agq_num_blocks(n, block))
    npk = int(L.lib.agq_packed_bytes(n, bits))
    if len(data) < off + 4 * nb:
        raise L.ProtocolError("tensor dump: truncated input")
    if len(data) < off + 4 * nb + npk:
        raise L.ProtocolError("tensor dump: truncated codes")
    scales = torch.frombuffer(bytearray(data[off:off + 4 * nb]), dtype=torch.float32).to(device)
    codes = torch.frombuffer(bytearray(data[off + 4 * nb:off + 4 * nb + npk]),
                             dtype=torch.uint8).to(device)
    if not packed:
        codes = unpack_codes(codes, bits, n)
    return QuantizedTensor(codes, scales, bits, block, tuple(shape), CodecKind(codec), packed)
