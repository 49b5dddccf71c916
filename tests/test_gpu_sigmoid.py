"""Post-processing numerics at the decision boundaries (reference pipeline.py:266-294,
model.py:351-353).

The device computes sigmoid(x) = 1 / (1 + exp(-clip(x, -60, 60))) in the reference's operation
order with a CORRECTLY ROUNDED exp (postprocess.cu exp_cr).  The reference's NumPy exp is a
faithful (<= 1 ulp) SIMD implementation that is not correctly rounded, so a reported score can
differ from NumPy's by 1 ulp; these tests pin (1) the device value against a 50-digit decimal
evaluation, and (2) that no gate / ordering decision differs from the reference's NumPy code on
fp32-representable logits (the device path's logits are fp32) next to every threshold tested,
on exact threshold hits, and in the saturated region where sigmoid values tie."""

import math
from decimal import Decimal, getcontext

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_11441_b200 as D  # noqa: E402

getcontext().prec = 50


class _Raw:
    def __init__(self, boxes, scores, pres):
        self.boxes, self.score_logits, self.presence_logits = boxes, scores, pres
        self.batch = scores.shape[0]


def sigmoid_cr(x: float) -> float:
    """Correctly rounded exp (50 significant digits, then round-to-nearest), reference op order."""
    x = min(max(float(x), -60.0), 60.0)
    e = float(Decimal(-x).exp())
    return 1.0 / (1.0 + e)


def sigmoid_numpy(x):
    """The reference's own formula (model.py:351-353)."""
    return 1.0 / (1.0 + np.exp(-np.clip(x, -60.0, 60.0)))


def device_sigmoids(x: np.ndarray):
    """sigmoid of every x through the device post-processing kernel: one class per value with a
    single query (gates open, nothing to suppress) -> Detection.score; the same values as
    presence logits -> Detection.presence."""
    n = x.shape[0]
    boxes = np.tile(np.array([0.5, 0.5, 0.2, 0.2]), (n, 1, 1))
    dets = D.postprocess(_Raw(boxes, x[:, None], x[::-1].copy()), [f"c{i}" for i in range(n)],
                         D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0))
    assert len(dets) == n
    return np.array([d.score for d in dets]), np.array([d.presence for d in dets])[::-1]


def f32_neighbours(x: float, k: int = 24):
    v = np.float32(x)
    out = [v]
    lo = hi = v
    for _ in range(k):
        lo = np.nextafter(lo, np.float32(-np.inf))
        hi = np.nextafter(hi, np.float32(np.inf))
        out += [lo, hi]
    return np.array(out, dtype=np.float64)


THRESHOLDS = [0.5, 0.45, 0.3, 0.1, 0.9, 0.05, 0.123456789, 0.999, 1e-6]


def test_device_sigmoid_is_correctly_rounded():
    rng = np.random.default_rng(0)
    xs = [rng.uniform(-60, 60, 1500), rng.normal(0, 3, 1500), rng.uniform(18, 40, 300),
          np.array([0.0, -0.0, 60.0, -60.0, 61.0, -61.0, 1e-300, -1e-300, 700.0, -700.0, 36.7, 37.0])]
    for t in THRESHOLDS:
        xs.append(f32_neighbours(math.log(t / (1 - t)), 8))
    x = np.concatenate(xs)
    s_dev, p_dev = device_sigmoids(x)
    ref = np.array([sigmoid_cr(v) for v in x])
    np.testing.assert_array_equal(s_dev, ref)
    np.testing.assert_array_equal(p_dev, ref)
    # and within 2 ulps of the reference's NumPy value everywhere: NumPy's exp is faithful (<= 1 ulp),
    # and 1 / (1 + e) can turn one ulp of e into two ulps of the quotient across a binade boundary
    npy = sigmoid_numpy(x)
    ulps = np.abs(s_dev - npy) / np.spacing(np.maximum(np.maximum(np.abs(npy), np.abs(s_dev)), 1e-300))
    assert ulps.max() <= 2.0, ulps.max()
    print(f"device == correctly rounded on {x.size} logits; NumPy differs by 1 ulp on "
          f"{int((s_dev != npy).sum())} of them")


@pytest.mark.parametrize("thr", THRESHOLDS)
def test_score_gate_next_to_threshold_matches_reference(thr):
    """fp32 logits within +-24 fp32 ulps of logit(thr): the inclusive score gate (pipeline.py:284)
    and the exclusive presence gate (pipeline.py:278) decide exactly like the reference's NumPy
    code (oracle restatement, pinned to the reference)."""
    from oracle import dart_oracle as O

    x = f32_neighbours(math.log(thr / (1 - thr)))
    n = x.shape[0]
    # one class per logit (score gate), and the same logits as presence logits (presence gate)
    boxes = np.tile(np.array([0.5, 0.5, 0.2, 0.2]), (n, 1, 1))
    cfg = D.PipelineConfig(presence_threshold=thr, score_threshold=thr)
    names = [f"c{i}" for i in range(n)]
    got = D.postprocess(_Raw(boxes, x[:, None], x.copy()), names, cfg)
    ref = O.postprocess(boxes, x[:, None], x.copy(), presence_thr=thr, score_thr=thr)
    assert [d.class_id for d in got] == [r[0] for r in ref]
    np_s = sigmoid_numpy(x)
    assert sum(np_s >= thr) == len(ref)  # both gates pass exactly where NumPy's sigmoid >= thr


def test_exact_threshold_hits():
    """sigmoid(0) = 0.5 exactly on every exp implementation: a 0.5 score gate keeps it (>=), a
    0.5 presence gate does not skip it (p < thr is false)."""
    box = [0.5, 0.5, 0.2, 0.2]
    cfg = D.PipelineConfig(presence_threshold=0.5, score_threshold=0.5)
    d = D.postprocess(_Raw(np.array([[box]]), np.array([[0.0]]), np.array([0.0])), ["car"], cfg)
    assert len(d) == 1 and d[0].score == 0.5 and d[0].presence == 0.5
    nudge = np.nextafter(0.0, -1.0)  # the smallest negative logit: sigmoid rounds to 0.5 too
    d = D.postprocess(_Raw(np.array([[box]]), np.array([[nudge]]), np.array([nudge])), ["car"], cfg)
    assert len(d) == 1 and sigmoid_numpy(nudge) == 0.5
    d = D.postprocess(_Raw(np.array([[box]]), np.array([[-1e-9]]), np.array([10.0])), ["car"], cfg)
    assert d == [] and sigmoid_numpy(-1e-9) < 0.5


@pytest.mark.parametrize("lo,hi", [(18.0, 37.0), (36.0, 80.0), (-3.0, 3.0)])
def test_saturated_ties_order_like_reference(lo, hi):
    """Sigmoid values tie in float64 well before the 60 clip (exactly 1.0 above ~36.7, a handful
    of distinct values in 18..37): ties must order by query index (pipeline.py:286).  200 fp32
    logits, disjoint boxes (no suppression): the kept order equals the reference's."""
    from oracle import dart_oracle as O

    rng = np.random.default_rng(int(abs(lo) * 10))
    Q = 200
    x = rng.uniform(lo, hi, (1, Q)).astype(np.float32).astype(np.float64)
    x[0, ::7] = x[0, 3]  # exact duplicates too
    g = np.arange(Q)
    boxes = np.stack([(g % 20) / 20 + 0.025, (g // 20) / 10 + 0.05, np.full(Q, 0.02), np.full(Q, 0.02)], -1)[None]
    cfg = D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0)
    got = D.postprocess(_Raw(boxes, x, np.array([10.0])), ["car"], cfg)
    ref = O.postprocess(boxes, x, np.array([10.0]), presence_thr=0.0, score_thr=0.0)
    assert [d.query for d in got] == [r[1] for r in ref]
    assert len(got) == Q
    ties = len(ref) - len({r[3] for r in ref})
    print(f"[{lo},{hi}]: {ties} tied scores, order identical")
