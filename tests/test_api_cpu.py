"""Host-side API mirror (CPU): config invariants, bit-exact deterministic init against the
reference's fixtures, scenes, text rows, serialization, pipeline config."""

import json

import numpy as np
import pytest

import paper_2603_11441_b200 as D
from conftest import load_golden
from paper_2603_11441_b200.model import _text_rows


@pytest.mark.parametrize("name", ["A", "A2", "B", "C"])
def test_init_bit_exact_vs_reference(name):
    g = load_golden(name)
    cfg = D.ModelConfig.from_dict(json.loads(str(g["config_json"])))
    if cfg.num_blocks > 8:  # full ViT-H: check the enc-dec + a sample of blocks to stay fast
        m = D.build_model(cfg, with_mask_head=False)
    else:
        m = D.build_model(cfg, with_mask_head=False)
    assert list(m.params) == [str(n) for n in g["param_names"]]
    assert D.weights_checksum(m) == str(g["weights_checksum"])


def test_scene_and_text_rows_match_reference():
    g = load_golden("A")
    img, _ = D.generate_scene(D.SceneSpec(seed=1, num_classes=3))
    np.testing.assert_array_equal(img.astype(np.float32), g["image"])
    assert [_text_rows(str(n), 8) for n in g["names"]] == g["text_rows"].tolist()


def test_config_invariants():
    with pytest.raises(D.ConfigError):
        D.toy_config(global_block_indices=()).validate()
    with pytest.raises(D.ConfigError):
        D.toy_config(image_size=60).validate()
    with pytest.raises(D.ConfigError):
        D.toy_config(window_size=3).validate()
    cfg = D.toy_config(seed=5)
    assert D.ModelConfig.from_dict(cfg.to_dict()) == cfg
    D.vit_h_config().validate()
    assert D.vit_h_config().tokens == 5184 and D.vit_h_config().head_dim == 80


def test_serialization_roundtrip(tmp_path):
    m = D.build_model(D.toy_config(seed=1), with_mask_head=False)
    p = tmp_path / "m.dartm"
    D.save_model(m, p)
    m2 = D.load_model(p)
    assert D.models_equal(m, m2)


def test_text_cache_semantics():
    m = D.build_model(D.toy_config(), with_mask_head=False)
    a = D.text_encode(m, ["car"]).by_name["car"]
    assert D.text_encode(m, ["car"]).by_name["car"] is a
    with pytest.raises(ValueError):
        D.text_encode(m, [""])
    with pytest.raises(ValueError):
        D.text_encode(m, [])


def test_structural_edits():
    m = D.build_model(D.toy_config(), with_mask_head=False)
    t = D.truncate_model(m, 2)
    assert t.block_kinds == ("windowed", "global") and t.config.num_blocks == 2
    s = D.set_sub_block(m, 0, "attn", False)
    assert s.attn_enabled[0] is False and m.attn_enabled[0] is True


def test_pipeline_config_and_levels():
    with pytest.raises(ValueError):
        D.PipelineConfig(n_max=0)
    with pytest.raises(ValueError):
        D.PipelineConfig(score_threshold=1.5)
    cfg = D.PipelineConfig.for_level(D.PipelineLevel.BATCHED_DET_ONLY_FP16)
    assert cfg.detection_only and cfg.backbone_mode is D.PrecisionMode.FP16_ACCUM_FP32
    assert D.chunk_count(80, 16) == 5 and D.chunk_count(10, 4) == 3 and D.chunk_count(7, None) == 1
    d = D.Detection(0, "car", (0.1, 0.2, 0.3, 0.4), 0.55, 0.66, 3)
    assert D.detections_from_json(D.detections_to_json([d])) == [d]


def test_host_iou_matches_oracle():
    from oracle import dart_oracle as O

    rng = np.random.default_rng(0)
    for _ in range(200):
        a, b = rng.uniform(0, 1, 4), rng.uniform(0, 1, 4)
        assert D.box_iou(a, b) == O.box_iou(a, b)


def test_fpn_features_host_arrays_and_finiteness():
    """Reference model.py:152-166: FpnFeatures built from host arrays (as distill.py:109-113 does)
    exposes float64 `.levels`, and any non-finite level raises ValueError at construction."""
    import paper_2603_11441_b200 as D

    lv = (np.ones((16, 8), np.float32), np.zeros((4, 8)), np.full((1, 8), 2.0))
    f = D.FpnFeatures(lv, 0, D.PrecisionMode.FP32)
    assert all(a.dtype == np.float64 for a in f.levels)
    np.testing.assert_array_equal(f.levels[0], np.ones((16, 8)))
    for bad in (np.nan, np.inf, -np.inf):
        b = lv[1].copy()
        b[0, 0] = bad
        with pytest.raises(ValueError, match="finite"):
            D.FpnFeatures((lv[0], b, lv[2]), 0, D.PrecisionMode.FP32)
    with pytest.raises(ValueError):
        D.FpnFeatures(lv[:2], 0, D.PrecisionMode.FP32)
