"""Mask head (the non-detection-only path, reference model.py:573-579)
against the reference's own outputs (tests/golden/golden_M.npz, oracle/make_golden.py M)."""

import json

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_11441_b200 as D  # noqa: E402


def _model(g):
    cfg = D.ModelConfig.from_dict(json.loads(str(g["config_json"])))
    m = D.build_model(cfg, with_mask_head=True)
    assert D.weights_checksum(m) == str(g["weights_checksum"])
    return m


class _Raw:  # the reference's raw outputs (float64 host)
    def __init__(self, qf):
        self.query_features = qf
        self.d_query_features = None


class _Fpn:
    def __init__(self, l0):
        self.levels = (l0, None, None)


def test_mask_head_on_reference_inputs():
    """Device mask GEMMs on the reference's L0 / query features: fp16 operands, fp32
    accumulation; max error <= 1% of the largest |logit|."""
    g = load_golden("M")
    m = _model(g)
    got = D.mask_head_forward(m, _Fpn(g["L0"]), _Raw(g["query_features"]))
    ref = g["masks"]
    assert got.shape == ref.shape and got.dtype == np.float64
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-2, err


def test_mask_head_end_to_end():
    """Our backbone + enc-dec + mask head vs the reference's full path (toy config)."""
    g = load_golden("M")
    m = _model(g)
    names = [str(n) for n in g["names"]]
    fpn = D.backbone_forward(m, g["image"].astype(np.float64))
    raw = D.encdec_forward(m, fpn, D.text_encode(m, names).stack(names))
    got = D.mask_head_forward(m, fpn, raw)
    ref = g["masks"]
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 3e-2, err


def test_pipeline_levels_with_mask_head():
    """NAIVE / SHARED levels (detection_only=False) run the mask head once per enc-dec pass and
    return the same detections as the batched detection-only level (reference
    tests/test_acceptance.py:67-90)."""
    g = load_golden("M")
    m = _model(g)
    names = [str(n) for n in g["names"]]
    image = g["image"].astype(np.float64)
    thr = dict(presence_threshold=0.0, score_threshold=0.0)
    c = D.RunCounters()
    naive = D.run_naive(m, image, names, D.PipelineConfig(detection_only=False, **thr), c)
    assert c.mask_head_calls == len(names)
    ref = D.run_batched(m, image, names, D.PipelineConfig(**thr))
    assert naive == ref
    with pytest.raises(D.MaskHeadRemovedError):
        D.mask_head_forward(D.without_mask_head(m), None, None)
