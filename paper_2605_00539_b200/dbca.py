"""L2b control plane: the DBCA per-stage bit-width policy (dbca.hpp:13-177)
and the activation-storage policy (layers.hpp:15-93, 148-177, 266-301).

The planner arithmetic runs in the C++ library (agq_plan_bit_widths); this
module mirrors the reference's types. `ActivationStore` is the layer-aware
activation quantizer: it stores the tensors a transformer block keeps for
backward under `agoq_default(bits)` and quantizes them with one grouped
sm_100a launch per stage.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Dict

import torch

from . import _lib as L
from .codec import (CodecKind, ErrorRecord, QuantizedTensor, dequantize_grouped,
                    quantize_grouped)


@dataclass
class PipelineConfig:  # dbca.hpp:13-29
    n_stages: int = 1
    micro_batches: int = 8
    interleave: int = 2


def stored_activation_counts(cfg: PipelineConfig) -> list:
    """dbca.hpp:34-41: device d of n holds 3n - 2d + 1 micro-batches."""
    arr = (C.c_int * max(cfg.n_stages, 1))()
    L.check(L.lib.agq_stored_activation_counts(cfg.n_stages, cfg.micro_batches, cfg.interleave,
                                               arr))
    return [int(v) for v in arr[: cfg.n_stages]]


@dataclass
class StagePlan:  # dbca.hpp:43-48
    stage_index: int
    stored_minibatches: int
    raw_bits: float
    assigned_bits: int


@dataclass
class BitWidthPlan:  # dbca.hpp:50-59
    n_stages: int
    stages: list

    def assigned(self) -> list:
        return [s.assigned_bits for s in self.stages]


def plan_bit_widths(cfg: PipelineConfig) -> BitWidthPlan:
    """dbca.hpp:63-78: B_i = clamp(lround(4 N_max / N_i), 4, 8)."""
    n = max(cfg.n_stages, 1)
    counts, raw, bits = (C.c_int * n)(), (C.c_double * n)(), (C.c_int * n)()
    L.check(L.lib.agq_plan_bit_widths(cfg.n_stages, cfg.micro_batches, cfg.interleave, counts,
                                      raw, bits))
    return BitWidthPlan(cfg.n_stages, [StagePlan(i + 1, counts[i], raw[i], bits[i])
                                       for i in range(cfg.n_stages)])


@dataclass
class PeakMemoryCheck:  # dbca.hpp:86-93
    stages: list
    budget_bytes: float
    slack_bytes: float
    passed: bool


def peak_memory_check(plan: BitWidthPlan, bytes_per_minibatch_at_16bit: float) -> PeakMemoryCheck:
    """dbca.hpp:98-124."""
    if not plan.stages:
        raise L.InvalidArgument("empty plan")
    unit = bytes_per_minibatch_at_16bit / 16.0
    n_max = max(s.stored_minibatches for s in plan.stages)
    budget = n_max * 4.0 * unit
    ok, rows, max_slack = True, [], 0.0
    for s in plan.stages:
        b = s.stored_minibatches * float(s.assigned_bits) * unit
        slack = s.stored_minibatches * 1.0 * unit
        max_slack = max(max_slack, slack)
        ok = ok and not (b > budget + slack)
        rows.append({"stage": s.stage_index, "bytes": b, "budget_bytes": budget + slack})
    return PeakMemoryCheck(rows, budget, max_slack, ok)


def plan_reuse_check(low: PipelineConfig, high: PipelineConfig):
    """dbca.hpp:139-168: applies a smaller pipeline's plan to a larger one."""
    if low.n_stages > high.n_stages:
        raise L.InvalidArgument("plan reuse goes from fewer stages to more stages")
    lp = plan_bit_widths(low)
    hc = stored_activation_counts(high)
    applied = [4] * len(hc)
    for i in range(low.n_stages):
        applied[len(hc) - 1 - i] = lp.stages[low.n_stages - 1 - i].assigned_bits
    peak = max(c * b for c, b in zip(hc, applied))
    u4 = max(c * 4.0 for c in hc)
    ok = all(not (c * b > u4 + c) for c, b in zip(hc, applied))
    return {"applied_bits": applied, "peak": float(peak), "uniform4_peak": u4, "pass": ok}


class LayerRole(enum.Enum):  # layers.hpp:15-23
    RmsNorm = "rmsnorm"
    QkvProj = "qkv_proj"
    Attention = "attention"
    OutProj = "out_proj"
    Ffn1 = "ffn1"
    SiluMul = "silu_mul"
    Ffn2 = "ffn2"


class SaveStrategy(enum.Enum):  # layers.hpp:37-41
    RecomputeIntermediates = 0
    CacheIntermediates = 1
    NoQuant = 2


@dataclass
class PolicyEntry:
    bit_width: int = 0  # 0 = full precision
    strategy: SaveStrategy = SaveStrategy.NoQuant


@dataclass
class ActivationPolicy:  # layers.hpp:48-93
    entries: Dict[LayerRole, PolicyEntry] = field(default_factory=dict)

    @staticmethod
    def all_full() -> "ActivationPolicy":
        return ActivationPolicy({r: PolicyEntry(0, SaveStrategy.NoQuant) for r in LayerRole})

    @staticmethod
    def agoq_default(bits: int = 4) -> "ActivationPolicy":
        R, S = LayerRole, SaveStrategy
        p = ActivationPolicy({
            R.RmsNorm: PolicyEntry(bits, S.RecomputeIntermediates),
            R.QkvProj: PolicyEntry(bits, S.RecomputeIntermediates),
            R.Attention: PolicyEntry(0, S.NoQuant),
            R.OutProj: PolicyEntry(bits, S.CacheIntermediates),
            R.Ffn1: PolicyEntry(bits, S.RecomputeIntermediates),
            R.SiluMul: PolicyEntry(bits, S.RecomputeIntermediates),
            R.Ffn2: PolicyEntry(bits, S.RecomputeIntermediates),
        })
        p.validate()
        return p

    def at(self, role: LayerRole) -> PolicyEntry:
        if role not in self.entries:
            raise RuntimeError(f"policy has no entry for role {role.value}")
        return self.entries[role]

    def validate(self):
        for e in self.entries.values():
            if e.bit_width != 0 and not (4 <= e.bit_width <= 8):
                raise L.InvalidArgument("policy bit width must be FULL or in [4,8]")
            if e.strategy == SaveStrategy.NoQuant and e.bit_width != 0:
                raise L.InvalidArgument("NO_QUANT entries store full precision")


def stage_policy(plan: BitWidthPlan, stage_index: int) -> ActivationPolicy:
    """dbca.hpp:172-177."""
    for s in plan.stages:
        if s.stage_index == stage_index:
            return ActivationPolicy.agoq_default(s.assigned_bits)
    raise L.InvalidArgument("no such stage in plan")


# Which role's entry governs each tensor a block stores for backward
# (layers.hpp:266-301 layer_forward): norm inputs by RmsNorm, the out-proj
# input by OutProj (cached, quantized), the SiLU&Mul inputs by SiluMul;
# Q/K/V follow Attention (full precision).
STORED_TENSORS = {
    "norm1_input": LayerRole.RmsNorm,
    "norm2_input": LayerRole.RmsNorm,
    "outproj_input": LayerRole.OutProj,
    "silu_gate": LayerRole.SiluMul,
    "silu_value": LayerRole.SiluMul,
    "q": LayerRole.Attention,
    "k": LayerRole.Attention,
    "v": LayerRole.Attention,
}


class ActivationStore:
    """SavedActivations (layers.hpp:180-192) on device: store() quantizes the
    policy's tensors (one grouped launch per distinct width), read() returns
    the dequantized tensor (bf16 by default)."""

    def __init__(self, policy: ActivationPolicy):
        policy.validate()
        self.policy = policy
        self.entries: Dict[str, object] = {}

    def store(self, tensors: Dict[str, torch.Tensor], stream=None, check: bool = True,
              errors: ErrorRecord | None = None):
        by_bits: Dict[int, list] = {}
        for name, t in tensors.items():
            e = self.policy.at(STORED_TENSORS[name])
            if e.bit_width == 0:
                self.entries[name] = t
            else:
                by_bits.setdefault(e.bit_width, []).append(name)
        for bits, names in by_bits.items():
            qs = quantize_grouped([tensors[n] for n in names], bits, CodecKind.SymmetricLinear,
                                  stream=stream, check=check, errors=errors)
            for n, q in zip(names, qs):
                self.entries[n] = q

    def has(self, name: str) -> bool:
        return name in self.entries

    def read(self, name: str, out_dtype: torch.dtype = torch.bfloat16, stream=None):
        if name not in self.entries:
            raise RuntimeError(f"saved activations: missing tensor '{name}' required by the policy")
        e = self.entries[name]
        if isinstance(e, QuantizedTensor):
            return dequantize_grouped([e], out_dtype, stream=stream)[0]
        return e

    def nbytes(self) -> int:
        tot = 0
        for e in self.entries.values():
            tot += e.nbytes() if isinstance(e, QuantizedTensor) else e.numel() * e.element_size()
        return tot


class StageActivationStore:
    """Every layer's SavedActivations (layers.hpp:180-192, stored set
    :266-301) of one pipeline stage under the stage's policy
    (dbca.hpp:172-177 stage_policy): store() quantizes the quantized tensors
    of ALL layers in one grouped launch per width (LLaMA-8B at 8 stages: 4
    layers x 5 tensors = 20 tensors, one launch); read_all() dequantizes them
    back in one grouped launch with the reference's validate checks."""

    def __init__(self, policy: ActivationPolicy):
        policy.validate()
        self.policy = policy
        self.layers: list = []

    def store(self, layers, stream=None, check: bool = True, errors: ErrorRecord | None = None):
        self.layers = [dict() for _ in layers]
        by_bits: Dict[int, list] = {}
        for li, tensors in enumerate(layers):
            for name, t in tensors.items():
                e = self.policy.at(STORED_TENSORS[name])
                if e.bit_width == 0:
                    self.layers[li][name] = t
                else:
                    by_bits.setdefault(e.bit_width, []).append((li, name))
        for bits, keys in by_bits.items():
            qs = quantize_grouped([layers[li][n] for li, n in keys], bits,
                                  CodecKind.SymmetricLinear, stream=stream, check=check,
                                  errors=errors)
            for (li, n), q in zip(keys, qs):
                self.layers[li][n] = q

    def read(self, layer: int, name: str, out_dtype: torch.dtype = torch.bfloat16, stream=None):
        if layer >= len(self.layers) or name not in self.layers[layer]:
            raise RuntimeError(f"saved activations: missing tensor '{name}' required by the policy")
        e = self.layers[layer][name]
        if isinstance(e, QuantizedTensor):
            return dequantize_grouped([e], out_dtype, stream=stream)[0]
        return e

    def read_all(self, out_dtype: torch.dtype = torch.bfloat16, stream=None, check: bool = True):
        out = [dict() for _ in self.layers]
        by_bits: Dict[int, list] = {}
        for li, d in enumerate(self.layers):
            for name, e in d.items():
                if isinstance(e, QuantizedTensor):
                    by_bits.setdefault(e.bit_width, []).append((li, name))
                else:
                    out[li][name] = e
        for bits, keys in by_bits.items():
            ts = dequantize_grouped([self.layers[li][n] for li, n in keys], out_dtype,
                                    stream=stream, check=check)
            for (li, n), t in zip(keys, ts):
                out[li][n] = t
        return out

    def nbytes(self) -> int:
        tot = 0
        for d in self.layers:
            for e in d.values():
                tot += e.nbytes() if isinstance(e, QuantizedTensor) else e.numel() * e.element_size()
        return tot
