"""paper_2603_11441_b200 -- a B200-native (sm_100a) implementation of DART's multi-class
detection path (arXiv 2603.11441): one class-agnostic ViT backbone pass per image, one
class-batched 6+6-layer encoder-decoder, box/score/presence heads and detection-only
post-processing, behind the reference's Python detector API (`dart.model` /
`dart.pipeline`).  All arithmetic runs in libdart_b200.so (include/dart_b200.h)."""

__version__ = "0.1.0"

from .model import (  # noqa: F401
    ConfigError,
    DetectorModel,
    FpnFeatures,
    MaskHeadRemovedError,
    ModelConfig,
    RawQueryOutputs,
    TextEmbeddings,
    backbone_forward,
    build_model,
    clear_text_cache,
    encdec_forward,
    load_model,
    mask_head_forward,
    mask_head_forward_device,
    models_equal,
    save_model,
    set_sub_block,
    sigmoid,
    text_encode,
    toy_config,
    truncate_model,
    vit_h_config,
    weights_checksum,
    without_mask_head,
)
from .pipeline import (  # noqa: F401
    Detection,
    EmptyClassSetError,
    PipelineConfig,
    PipelineLevel,
    PrecisionStudyReport,
    RunCounters,
    box_iou,
    chunk_count,
    detections_from_json,
    detections_to_json,
    postprocess,
    precision_study,
    run_batched,
    run_batched_from_fpn,
    run_level,
    run_naive,
    run_shared,
)
from .scenes import SceneSpec, generate_scene, scene_images  # noqa: F401
from .tensors import PrecisionMode, ShapeError, cosine_similarity  # noqa: F401
