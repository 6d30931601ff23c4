"""Synthetic inputs with the reference's bytes.

tools/agq.cpp:47-65 InputSpec::materialize draws every CLI input from
make_rng(seed, 0x1D) (rng.hpp:9-28: std::mt19937_64 seeded by derive_seed)
through std::normal_distribution<float>(0, 1) (or uniform / constant);
all-reduce worker r uses seed + r (agq.cpp:279). agq_fill_input
(capi.cpp) runs the same libstdc++ engine and distributions on the host, so
a tensor made here holds exactly the reference's values. Host-side input
synthesis only: the data path consumes the tensor wherever it is copied to.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib as L

KINDS = {"normal": 0, "uniform": 1, "const": 2}
REF_STREAM = 0x1D  # agq.cpp:55


def materialize(n: int, seed: int, kind: str = "normal", a: float = 0.0, b: float = 1.0,
                dtype: torch.dtype = torch.float32, stream: int = REF_STREAM, index: int = 0,
                pin: bool = False, out: torch.Tensor | None = None) -> torch.Tensor:
    """n values from make_rng(seed, stream, index): normal(a, b), uniform(a, b)
    or the constant a, as float32 or their bfloat16 round-to-nearest-even.
    Returns a CPU tensor (pinned if asked) or fills `out` (CPU, contiguous)."""
    if dtype not in (torch.float32, torch.bfloat16):
        raise L.InvalidArgument("inputs are float32 or bfloat16")
    if out is None:
        out = torch.empty(int(n), dtype=dtype, pin_memory=pin)
    elif out.is_cuda or not out.is_contiguous() or out.numel() != n or out.dtype != dtype:
        raise L.InvalidArgument("out must be a contiguous CPU tensor of n values")
    L.check(L.lib.agq_fill_input(seed & (2**64 - 1), stream, index, KINDS[kind], float(a),
                                 float(b), L.AGQ_BF16 if dtype == torch.bfloat16 else L.AGQ_F32,
                                 out.data_ptr(), int(n)))
    return out


def materialize_parallel(sizes, seed: int, dtype: torch.dtype = torch.bfloat16, a: float = 0.0,
                         b: float = 1.0, scales=None, pin: bool = False, stream: int = REF_STREAM):
    """One tensor per entry of `sizes`, tensor i from make_rng(seed, stream,
    index=i) (independent sub-streams, drawn on parallel host threads; the
    ctypes call releases the GIL). scales[i] multiplies normal tensor i's
    standard deviation."""
    from concurrent.futures import ThreadPoolExecutor
    outs = [torch.empty(int(n), dtype=dtype, pin_memory=pin) for n in sizes]

    def one(i):
        sd = b * (scales[i] if scales else 1.0)
        materialize(sizes[i], seed, "normal", a, sd, dtype, stream, i, out=outs[i])

    with ThreadPoolExecutor(max_workers=max(1, len(sizes))) as ex:
        list(ex.map(one, range(len(sizes))))
    return outs
