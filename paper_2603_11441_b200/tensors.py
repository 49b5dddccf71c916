"""Precision tags and shape errors of the detector API (reference tensors.py:29-42).

The B200 path implements ONE arithmetic discipline: fp16 GEMM/attention operands with
fp32 tensor-core accumulation, fp32 residual streams, fp32 LayerNorm / softmax / RoPE,
fp64 post-processing decisions.  It is recorded as `DEVICE_FP16_ACCUM_FP32`; requests
for FP32 or FP16_ACCUM_FP32 run it, FP16_ACCUM_FP16 (the reference's failure-mode
emulation) is rejected.
"""

from __future__ import annotations

from enum import Enum


class ShapeError(ValueError):
    """Operand shapes are incompatible for the requested operation (tensors.py:29)."""


class PrecisionMode(Enum):
    FP32 = "fp32"
    FP16_ACCUM_FP32 = "fp16-accum-fp32"
    FP16_ACCUM_FP16 = "fp16-accum-fp16"
    DEVICE_FP16_ACCUM_FP32 = "device-fp16-accum-fp32"

    @property
    def is_half(self) -> bool:
        return self is not PrecisionMode.FP32


def device_mode(requested: PrecisionMode) -> PrecisionMode:
    """The discipline actually run for a requested mode."""
    if requested is PrecisionMode.FP16_ACCUM_FP16:
        raise ValueError("FP16_ACCUM_FP16 is a failure-mode emulation; the B200 path accumulates in fp32")
    return PrecisionMode.DEVICE_FP16_ACCUM_FP32
