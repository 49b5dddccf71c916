"""RunCounters semantics of the drop-in pipeline API on the GPU path: a port of the reference's
TestCounters (tests/test_pipeline.py:77-121; counters pipeline.py:112-122, 134-154), plus the
level-equivalence tests around them (tests/test_pipeline.py:33-66)."""

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_11441_b200 as D  # noqa: E402
from paper_2603_11441_b200.pipeline import PipelineLevel  # noqa: E402

NAMES = ["car", "person", "dog"]


def det_cfg(**over):
    return D.PipelineConfig.for_level(PipelineLevel.BATCHED_DET_ONLY, **over)


@pytest.fixture(scope="module")
def toy_model():
    return D.build_model(D.toy_config(seed=0))


@pytest.fixture(scope="module")
def sample_image():
    return D.generate_scene(D.SceneSpec(seed=1, num_classes=3))[0]


def test_naive_runs_backbone_per_class(toy_model, sample_image):
    c = D.RunCounters()
    D.run_naive(toy_model, sample_image, NAMES, det_cfg(), c)
    assert c.backbone_passes == 3
    assert c.encdec_passes == 3


def test_shared_runs_backbone_once(toy_model, sample_image):
    c = D.RunCounters()
    D.run_shared(toy_model, sample_image, NAMES, det_cfg(), c)
    assert c.backbone_passes == 1
    assert c.encdec_passes == 3


def test_batched_chunking(toy_model, sample_image):
    names = [f"class{i:02d}" for i in range(10)]
    c = D.RunCounters()
    D.run_batched(toy_model, sample_image, names, det_cfg(n_max=4), c)
    assert c.backbone_passes == 1
    assert c.encdec_passes == 3
    assert c.encdec_classes == 10


def test_chunk_count_arithmetic():
    assert D.chunk_count(80, 16) == 5
    assert D.chunk_count(10, 4) == 3
    assert D.chunk_count(1, 1) == 1
    assert D.chunk_count(7, None) == 1


def test_detection_only_never_calls_mask_head(toy_model, sample_image):
    c = D.RunCounters()
    D.run_batched(toy_model, sample_image, NAMES, det_cfg(), c)
    assert c.mask_head_calls == 0


def test_mask_head_counts_when_enabled(toy_model, sample_image):
    c = D.RunCounters()
    D.run_shared(toy_model, sample_image, NAMES, det_cfg(detection_only=False), c)
    assert c.mask_head_calls == 3


def test_text_cache_hits(sample_image):
    model = D.build_model(D.toy_config(seed=3))
    c = D.RunCounters()
    D.run_batched(model, sample_image, ["car", "person"], det_cfg(), c)
    assert c.text_cache_misses == 2 and c.text_cache_hits == 0
    c2 = D.RunCounters()
    D.run_batched(model, sample_image, ["car", "person"], det_cfg(), c2)
    assert c2.text_cache_hits == 2 and c2.text_cache_misses == 0


def test_counters_as_dict_and_run_level(toy_model, sample_image):
    c = D.RunCounters()
    cfg = D.PipelineConfig.for_level(PipelineLevel.NAIVE)
    D.run_level(toy_model, sample_image, NAMES, cfg, c)
    d = c.as_dict()
    assert d["backbone_passes"] == 3 and d["encdec_passes"] == 3 and d["encdec_classes"] == 3
    assert d["mask_head_calls"] == 3  # NAIVE keeps the mask head (pipeline.py:94-99)


def test_levels_bitwise_equal_with_and_without_mask_head(toy_model, sample_image):
    cfg = det_cfg()
    naive = D.run_naive(toy_model, sample_image, NAMES, cfg)
    assert naive == D.run_shared(toy_model, sample_image, NAMES, cfg) == D.run_batched(toy_model, sample_image,
                                                                                          NAMES, cfg)
    cfg = det_cfg(detection_only=False)
    assert D.run_naive(toy_model, sample_image, NAMES, cfg) == D.run_batched(toy_model, sample_image, NAMES, cfg)


def test_empty_class_set_rejected(toy_model, sample_image):
    with pytest.raises(D.EmptyClassSetError):
        D.run_shared(toy_model, sample_image, [], det_cfg())
    with pytest.raises(D.EmptyClassSetError):
        D.run_batched(toy_model, sample_image, [], det_cfg())
