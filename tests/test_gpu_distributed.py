"""Class-sharded protocol on the real CUDA engine with a single-rank NCCL group (the
8-GPU run is not available here): output must equal run_batched bitwise."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_11441_b200 as D  # noqa: E402
from paper_2603_11441_b200.distributed import NativeEngine, detect_class_sharded  # noqa: E402


def test_single_rank_nccl_class_sharded_equals_batched():
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
        image, _ = D.generate_scene(D.SceneSpec(seed=1, num_classes=3))
        names = ["car", "person", "dog", "cat", "bus"]
        cfg = D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0)
        eng = NativeEngine(model)
        got = detect_class_sharded(eng, torch.from_numpy(image.astype(np.float32))[None].cuda(), names, cfg)
        assert got == D.run_batched(model, image, names, cfg)
    finally:
        dist.destroy_process_group()
