"""B200-native AGoQ quantization hot path (arXiv 2605.00539).

Drop-in for the reference's hot path (/root/reference/proj/include/agq):
block-wise activation quantize/dequantize at 4-8 bits under the DBCA
per-stage policy, fused FP8-E4M3 gradient accumulation, and the decomposed
precision-preserving 8-bit all-reduce. Everything runs in hand-written
sm_100a kernels of libagq_cuda.so behind a C ABI (include/agq_cuda.h);
the C++ drop-in headers live in include/agq_b200/.
"""
from . import _lib
from ._lib import CudaError, InvalidArgument, ProtocolError
from .codec import (CodecKind, ErrorRecord, QuantizedTensor, check_codec_args,
                    code_unit_value, dequantize_blockwise, dequantize_grouped, kDefaultBlockSize,
                    pack_codes, quantize_blockwise, quantize_grouped, quantize_roundtrip,
                    roundtrip_relative_delta,
                    unpack_codes, validate)
from .gradient import (AccumulatePrecision, ChunkAssignment, TraceEvent, allreduce_naive_simulated,
                       allreduce_simulated, decomposed_trace, local_accumulate, naive_trace,
                       round_bf16)
from .dbca import (ActivationPolicy, ActivationStore, BitWidthPlan, LayerRole, PipelineConfig,
                   PolicyEntry, SaveStrategy, StageActivationStore, peak_memory_check,
                   plan_bit_widths, plan_reuse_check,
                   stage_policy, stored_activation_counts)
from .scalar import fp4_decode, fp4_encode, fp8_decode, fp8_encode

__all__ = [n for n in dir() if not n.startswith("_")]


def launch_count() -> int:
    """Kernels launched by libagq_cuda.so in this process."""
    return int(_lib.lib.agq_launch_count())


def device_ok() -> bool:
    return bool(_lib.lib.agq_device_ok())
