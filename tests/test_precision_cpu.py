"""Host logic of the precision modes and the precision-study API (no GPU): mode mapping and
the reference's argument validation (pipeline.py:348-355)."""

import numpy as np
import pytest

import paper_2603_11441_b200 as D
from paper_2603_11441_b200.tensors import PrecisionMode as PM, device_mode, precision_code


def test_device_mode_mapping():
    for m in (PM.FP32, PM.FP16_ACCUM_FP32, PM.DEVICE_FP16_ACCUM_FP32):
        assert device_mode(m) is PM.DEVICE_FP16_ACCUM_FP32
        assert precision_code(m) == 0
    assert precision_code(PM.DEVICE_FP16_STORAGE_ACCUM_FP32) == 1
    assert device_mode(PM.FP16_ACCUM_FP16, backbone=True) is PM.DEVICE_FP16_ACCUM_FP16
    assert precision_code(PM.FP16_ACCUM_FP16) == 2
    with pytest.raises(ValueError):
        device_mode(PM.FP16_ACCUM_FP16)  # the enc-dec accumulates in fp32 only
    with pytest.raises(ValueError):
        device_mode(PM.DEVICE_FP16_STORAGE_ACCUM_FP32)


def test_precision_study_validation():
    model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
    imgs = [np.zeros((64, 64, 3))] * 5
    with pytest.raises(ValueError, match="at least 5 images"):
        D.precision_study(model, imgs[:4], [1, 2, 3])
    with pytest.raises(ValueError, match="at least 3 depths"):
        D.precision_study(model, imgs, [1, 2])
    with pytest.raises(ValueError, match="exceeds num_blocks"):
        D.precision_study(model, imgs, [1, 2, 99])


def test_cosine_similarity_matches_reference_semantics():
    a = np.arange(1.0, 7.0).reshape(2, 3)
    assert D.cosine_similarity(a, 2 * a) == pytest.approx(1.0)
    assert D.cosine_similarity([1.0, 0.0], [0.0, 1.0]) == 0.0
    with pytest.raises(ValueError):
        D.cosine_similarity([0.0, 0.0], [1.0, 1.0])
    with pytest.raises(D.ShapeError):
        D.cosine_similarity([1.0], [1.0, 2.0])
