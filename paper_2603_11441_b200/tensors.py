"""Precision tags and shape errors of the detector API (reference tensors.py:29-42).

The detection path implements ONE arithmetic discipline: fp16 GEMM/attention operands with
fp32 tensor-core accumulation, fp32 residual streams, fp32 LayerNorm / softmax / RoPE,
fp64 post-processing decisions.  It is recorded as `DEVICE_FP16_ACCUM_FP32`; requests for
FP32 or FP16_ACCUM_FP32 run it.

For the precision study (reference pipeline.py:318-367) the backbone also
has two native degraded disciplines (dart_model_set_precision):
  DEVICE_FP16_STORAGE_ACCUM_FP32  fp16 storage: GEMM outputs and the residual stream rounded
                                  to fp16 after every add, fp32 accumulation;
  DEVICE_FP16_ACCUM_FP16          fp16 storage and fp16 tensor-core accumulation (the
                                  FP16_ACCUM_FP16 negative control; a request for
                                  FP16_ACCUM_FP16 runs it in the backbone).
The enc-dec always accumulates in fp32 and rejects FP16_ACCUM_FP16.
"""

from __future__ import annotations

from enum import Enum

import numpy as np


class ShapeError(ValueError):
    """Operand shapes are incompatible for the requested operation (tensors.py:29)."""


class PrecisionMode(Enum):
    FP32 = "fp32"
    FP16_ACCUM_FP32 = "fp16-accum-fp32"
    FP16_ACCUM_FP16 = "fp16-accum-fp16"
    DEVICE_FP16_ACCUM_FP32 = "device-fp16-accum-fp32"
    DEVICE_FP16_STORAGE_ACCUM_FP32 = "device-fp16-storage-accum-fp32"
    DEVICE_FP16_ACCUM_FP16 = "device-fp16-accum-fp16"

    @property
    def is_half(self) -> bool:
        return self is not PrecisionMode.FP32


# device discipline -> dart_model_set_precision code
_PRECISION_CODE = {
    PrecisionMode.DEVICE_FP16_ACCUM_FP32: 0,
    PrecisionMode.DEVICE_FP16_STORAGE_ACCUM_FP32: 1,
    PrecisionMode.DEVICE_FP16_ACCUM_FP16: 2,
}


def device_mode(requested: PrecisionMode, backbone: bool = False) -> PrecisionMode:
    """The discipline actually run for a requested mode (backbone=True: the backbone, which
    also implements the fp16-accumulation negative control)."""
    if requested in (PrecisionMode.FP16_ACCUM_FP16, PrecisionMode.DEVICE_FP16_ACCUM_FP16):
        if not backbone:
            raise ValueError("FP16_ACCUM_FP16 is a failure-mode emulation; the B200 enc-dec accumulates in fp32")
        return PrecisionMode.DEVICE_FP16_ACCUM_FP16
    if requested is PrecisionMode.DEVICE_FP16_STORAGE_ACCUM_FP32:
        if not backbone:
            raise ValueError("fp16-storage discipline is implemented for the backbone only")
        return requested
    return PrecisionMode.DEVICE_FP16_ACCUM_FP32


def precision_code(mode: PrecisionMode) -> int:
    return _PRECISION_CODE[device_mode(mode, backbone=True)]


def cosine_similarity(a, b) -> float:
    """Cosine of the angle between the flattened operands, float64 (tensors.py:260-270)."""
    av = np.asarray(a.detach().cpu().numpy() if hasattr(a, "detach") else a, dtype=np.float64).ravel()
    bv = np.asarray(b.detach().cpu().numpy() if hasattr(b, "detach") else b, dtype=np.float64).ravel()
    if av.shape != bv.shape:
        raise ShapeError(f"cosine_similarity shapes disagree: {av.shape} vs {bv.shape}")
    na = float(np.linalg.norm(av))
    nb = float(np.linalg.norm(bv))
    if na == 0.0 or nb == 0.0:
        raise ValueError("cosine similarity is undefined for a zero vector")
    return float(np.dot(av, bv) / (na * nb))
