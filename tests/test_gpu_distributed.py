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


def test_native_nccl_class_sharded_equals_encdec():
    """dart_class_sharded (the C ABI's own NCCL round, single-rank communicator): raw outputs of a
    2-image batch bitwise equal to dart_backbone + dart_encdec over the same classes, and the
    detections post-processed from them equal run_batched."""
    from paper_2603_11441_b200.distributed import NcclComm, class_sharded_raw_native

    model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
    imgs = [D.generate_scene(D.SceneSpec(seed=s, num_classes=3))[0] for s in (1, 2)]
    names = ["car", "person", "dog", "cat", "bus"]
    eng = NativeEngine(model)
    comm = NcclComm(1, 0)
    assert comm.lib.dart_nccl_comm_size(comm.ptr) == 1 and comm.lib.dart_nccl_comm_rank(comm.ptr) == 0
    x = torch.from_numpy(np.stack(imgs).astype(np.float32)).cuda()
    boxes, scores, pres, flags = class_sharded_raw_native(eng, comm, x, names)
    e1, fl = eng.prefix(x)
    rb, rs, rp = eng.decode(e1, names)
    torch.cuda.synchronize()
    assert int(flags.item()) == 0 and int(fl.item()) == 0
    assert torch.equal(boxes, rb) and torch.equal(scores, rs) and torch.equal(pres, rp)
    cfg = D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0)
    for b, img in enumerate(imgs):
        got = eng.postprocess(boxes[b].contiguous(), scores[b].contiguous(), pres[b].contiguous(), names, cfg)
        assert got == D.run_batched(model, img, names, cfg)
    comm.close()


def test_native_nccl_bad_image_flag():
    from paper_2603_11441_b200.distributed import NcclComm, class_sharded_raw_native

    model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
    image, _ = D.generate_scene(D.SceneSpec(seed=1, num_classes=3))
    image = image.copy()
    image[0, 0, 0] = 1.5  # outside [0, 1]
    eng = NativeEngine(model)
    comm = NcclComm(1, 0)
    _, _, _, flags = class_sharded_raw_native(eng, comm, torch.from_numpy(image.astype(np.float32))[None].cuda(),
                                              ["car", "dog"])
    with pytest.raises(ValueError):
        eng.check_flags(int(flags.item()))
    comm.close()


def test_native_nccl_failure_detection_and_abort():
    """SURVEY section 5 failure detection: a healthy communicator checks clean and a round awaited
    with a timeout completes; an aborted communicator reports the failure on every later call
    instead of blocking (no rank stays stuck in a collective)."""
    from paper_2603_11441_b200 import _native
    from paper_2603_11441_b200.distributed import NcclComm, class_sharded_raw_native

    model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
    image, _ = D.generate_scene(D.SceneSpec(seed=1, num_classes=3))
    x = torch.from_numpy(image.astype(np.float32))[None].cuda()
    eng = NativeEngine(model)
    comm = NcclComm(1, 0)
    comm.check()
    b0, s0, p0, f0 = class_sharded_raw_native(eng, comm, x, ["car", "dog"], timeout_s=60.0)
    assert int(f0.item()) == 0
    comm.abort()
    with pytest.raises(_native.NativeError):
        comm.check()
    with pytest.raises(_native.NativeError):
        class_sharded_raw_native(eng, comm, x, ["car", "dog"])
    comm.close()
