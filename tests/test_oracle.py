"""Pin the CPU oracle (oracle/dart_oracle.py) against fixtures produced by the real
reference (oracle/make_golden.py).  CPU only."""

import hashlib
import json

import numpy as np
import pytest

from conftest import load_golden
from oracle import dart_oracle as O


def cfg_from(g):
    d = json.loads(str(g["config_json"]))
    d["global_block_indices"] = tuple(d["global_block_indices"])
    d["fpn_dims"] = tuple(d["fpn_dims"])
    return O.OracleConfig(**d)


def _close(a, b, rtol=1e-10, atol=1e-12):
    np.testing.assert_allclose(a, b, rtol=rtol, atol=atol)


def dets_rows(dets):
    return np.array([[c, q, *box, s, p] for c, q, box, s, p in dets], dtype=np.float64).reshape(-1, 8)


@pytest.mark.parametrize("name", ["A", "A2"])
def test_weights_bit_exact(name):
    g = load_golden(name)
    cfg = cfg_from(g)
    P = O.build_params(cfg)
    names = [str(n) for n in g["param_names"]]
    assert names == [p for p, _, _ in O.param_declaration(cfg)]
    for n, h in zip(names, g["param_checksums"]):
        assert hashlib.blake2b(P[n].tobytes(), digest_size=8).hexdigest() == str(h), n
    assert O.weights_checksum(P) == str(g["weights_checksum"])


@pytest.mark.parametrize("name", ["A", "A2"])
def test_toy_end_to_end(name):
    g = load_golden(name)
    cfg = cfg_from(g)
    P = O.build_params(cfg)
    names = [str(n) for n in g["names"]]
    seed = {"A": 1, "A2": 5}[name]
    ncls = {"A": 3, "A2": 4}[name]
    image, _ = O.scene(seed, cfg.image_size, num_classes=ncls)
    assert hashlib.blake2b(image.tobytes(), digest_size=16).hexdigest() == str(g["image_checksum"])
    taps = {}
    l0, l1, l2 = O.backbone(P, cfg, image, taps)
    _close(taps["tokens"], g["tokens"])
    for b in range(cfg.num_blocks):
        _close(taps[f"block{b}"], g[f"block{b}"])
    _close(l0, g["L0"])
    _close(l1[g["L1_rows"]], g["L1"])
    _close(l2[g["L2_rows"]], g["L2"])
    assert [O.text_rows(n, cfg.text_tokens) for n in names] == g["text_rows"].tolist()
    texts = [O.text_embedding(P, cfg, n) for n in names]
    qf, boxes, pres, scores = O.encdec(P, cfg, l0, texts)
    _close(boxes, g["boxes"])
    _close(scores, g["score_logits"])
    _close(pres, g["presence_logits"])
    _close(qf[:, :8], g["qf_head"])
    # detections on the reference's own raw outputs must be identical
    for key in [k for k in g if k.startswith("dets_") and not k.endswith("_cfg")]:
        kw = json.loads(str(g[key + "_cfg"]))
        kw = {{"presence_threshold": "presence_thr", "score_threshold": "score_thr"}[k]: v for k, v in kw.items()}
        got = O.postprocess(g["boxes"], g["score_logits"], g["presence_logits"], cross_class=key.endswith("_xc"), **kw)
        np.testing.assert_array_equal(dets_rows(got), g[key])


def test_extra_class_list():
    g = load_golden("A")
    cfg = cfg_from(g)
    P = O.build_params(cfg)
    image, _ = O.scene(1, cfg.image_size, num_classes=3)
    l0, _, _ = O.backbone(P, cfg, image)
    names = [str(n) for n in g["list0_names"]]
    _, boxes, pres, scores = O.encdec(P, cfg, l0, [O.text_embedding(P, cfg, n) for n in names])
    _close(boxes, g["list0_boxes"])
    _close(scores, g["list0_score_logits"])
    _close(pres, g["list0_presence_logits"])


def test_postprocess_kats():
    """The reference's postprocess KATs (tests/test_pipeline.py:177-223)."""
    lg = lambda p: float(np.log(p / (1 - p)))
    box = [0.5, 0.5, 0.2, 0.2]
    d = O.postprocess(np.array([[box, box]]), np.array([[lg(0.9), lg(0.8)]]), np.array([10.0]))
    assert len(d) == 1 and abs(d[0][3] - 0.9) < 1e-12
    assert O.postprocess(np.array([[box]]), np.array([[lg(0.99)]]), np.array([-np.inf])) == []
    two = np.array([[[0.2, 0.2, 0.1, 0.1], [0.8, 0.8, 0.1, 0.1]]])
    assert len(O.postprocess(two, np.array([[lg(0.9), lg(0.8)]]), np.array([10.0]))) == 2
    assert O.postprocess(np.array([[box]]), np.array([[lg(0.3)]]), np.array([10.0])) == []
    a, b = [0.3, 0.3, 0.2, 0.2], [0.31, 0.3, 0.2, 0.2]
    d = O.postprocess(np.array([[b, a]]), np.array([[lg(0.8), lg(0.8)]]), np.array([10.0]))
    assert len(d) == 1 and d[0][1] == 0
    bb = np.array([[box], [box]])
    sc = np.array([[lg(0.9)], [lg(0.8)]])
    assert len(O.postprocess(bb, sc, np.array([10.0, 10.0]))) == 2
    d = O.postprocess(bb, sc, np.array([10.0, 10.0]), cross_class=True)
    assert len(d) == 1 and d[0][0] == 0
    assert O.box_iou(box, box) == pytest.approx(1.0)
    assert O.box_iou(box, (0.9, 0.9, 0.1, 0.1)) == 0.0


def test_patchify_validation():
    cfg = O.OracleConfig()
    with pytest.raises(ValueError):
        O.patchify(cfg, np.zeros((32, 32, 3)))
    with pytest.raises(ValueError):
        O.patchify(cfg, np.full((64, 64, 3), 1.5))


def test_rope_matches_complex_rotation():
    """RoPE as complex multiplication (reference tests/test_model.py:274-288)."""
    cfg = O.OracleConfig()
    cos, sin = O.rope_tables(cfg)
    x = np.random.default_rng(0).standard_normal((cfg.tokens, cfg.head_dim))
    z = (x[:, 0::2] + 1j * x[:, 1::2]) * (cos + 1j * sin)
    y = O.rope(x, cos, sin)
    np.testing.assert_allclose(y[:, 0::2], z.real, atol=1e-12)
    np.testing.assert_allclose(y[:, 1::2], z.imag, atol=1e-12)


def test_mask_head_matches_reference_golden():
    """Mask head restatement (model.py:573-579) vs the reference's own outputs (golden M):
    mask weights bit-exact, logits from the reference's L0 / query features to 1e-12."""
    g = load_golden("M")
    P = O.build_params(cfg_from(g), with_mask_head=True)
    got = [hashlib.blake2b(np.asarray(P[n], dtype=np.float64).tobytes(), digest_size=8).hexdigest()
           for n in ("mask.query_proj.w", "mask.query_proj.b", "mask.feat_proj.w", "mask.feat_proj.b")]
    assert got == [str(x) for x in g["mask_param_checksums"]]
    m = O.mask_head(P, g["L0"], g["query_features"])
    np.testing.assert_allclose(m, g["masks"], rtol=1e-12, atol=1e-12)
