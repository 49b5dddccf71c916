"""Inter-frame pipelining (two streams, two handles sharing the weights via dart_model_fork):
every image's detections are identical to the one-stream Detector.detect path, and forked
handles run the same kernels on the same weights (reference scheduler.py:128-187 models this
schedule; the outputs of a pipelined stream must equal per-frame detection)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_11441_b200 as D  # noqa: E402
from paper_2603_11441_b200.detector import Detector  # noqa: E402


def _setup(n_img=5):
    model = D.build_model(D.toy_config(seed=0), with_mask_head=False)
    names = ["car", "person", "dog"]
    cfg = D.PipelineConfig(presence_threshold=0.0, score_threshold=0.0)
    imgs = [D.generate_scene(D.SceneSpec(seed=10 + i, num_classes=3))[0].astype(np.float32) for i in range(n_img)]
    return model, names, cfg, imgs


@pytest.mark.parametrize("nbb", ["1", "2", "3"])
def test_detect_stream_matches_detect(nbb, monkeypatch):
    """1, 2 or 3 backbone streams (DART_PIPE_BB) taking images in turn: same detections."""
    monkeypatch.setenv("DART_PIPE_BB", nbb)
    model, names, cfg, imgs = _setup(7)
    det = Detector(model, names, cfg)
    serial = [det.detect(im) for im in imgs]
    streamed = [r[0] for r in det.detect_stream(imgs)]
    assert streamed == serial
    # device-resident pipelined path: image t's slot holds image t's results once its event fired
    outs = []
    for im in imgs:
        b, ev = det.detect_device_pipelined(torch.from_numpy(im[None]).cuda())
        ev.synchronize()
        outs.append(det.unpack({k: v.cpu() for k, v in det.result_tensors(b).items()}, 1)[0])
    assert outs == serial


def test_detect_stream_batched_and_device_inputs():
    model, names, cfg, imgs = _setup(6)
    det = Detector(model, names, cfg)
    batches = [np.stack(imgs[i:i + 2]) for i in range(0, 6, 2)]
    serial = [det.detect(b) for b in batches]
    dev = [torch.from_numpy(b).cuda() for b in batches]
    assert [r for r in det.detect_stream(dev)] == serial


def test_forked_handle_same_outputs():
    model, names, cfg, imgs = _setup(2)
    det = Detector(model, names, cfg)
    x = torch.from_numpy(np.stack(imgs[:1])).cuda()
    b = det.detect_device(x)
    ref = {k: v.clone() for k, v in det.result_tensors(b).items()}
    bp, ev = det.detect_device_pipelined(x)
    det.pipeline_join()
    torch.cuda.synchronize()
    got = det.result_tensors(bp)
    for k in ("flags", "kc", "pp", "boxes"):
        assert torch.equal(got[k], ref[k]), k
    for it, n in enumerate(ref["kc"].tolist()):  # kept lists (entries past the count are scratch)
        assert torch.equal(got["kq"][it, :n], ref["kq"][it, :n])
        assert torch.equal(got["ks"][it, :n], ref["ks"][it, :n])


def test_graph_pipeline_matches_detect():
    """CUDA-graph replay of the pipelined step: image t's detections (returned one step later)
    equal the eager one-stream path."""
    model, names, cfg, imgs = _setup(4)
    det = Detector(model, names, cfg)
    serial = []
    for im in imgs:
        b = det.detect_device(torch.from_numpy(im[None]).cuda())
        serial.append({k: v.clone() for k, v in det.result_tensors(b).items()})
    got = []
    for i, im in enumerate(imgs):
        b = det.detect_device_graph(torch.from_numpy(im[None]).cuda())
        if i > 0:
            got.append({k: v.clone() for k, v in det.result_tensors(b).items()})
    b = det.graph_drain()
    got.append({k: v.clone() for k, v in det.result_tensors(b).items()})
    torch.cuda.synchronize()
    for ref, g in zip(serial, got):
        for k in ("flags", "kc", "pp", "boxes"):
            assert torch.equal(g[k], ref[k]), k
        for it, n in enumerate(ref["kc"].tolist()):
            assert torch.equal(g["kq"][it, :n], ref["kq"][it, :n])


def test_stage_times_cover_the_step():
    """Detector.stage_times (CUDA events between backbone / enc-dec / post-processing, SURVEY section 5
    tracing): every stage is timed, the stages add up to the step, and the step still produces the
    same detections as detect()."""
    model, names, cfg, imgs = _setup(1)
    img = imgs[0]
    det = Detector(model, names, cfg)
    dimg = torch.from_numpy(img[None]).cuda()
    t = det.stage_times(dimg, reps=3)
    assert set(t) == {"backbone", "encdec", "postprocess", "total"}
    assert all(v > 0 for v in t.values())
    assert abs(t["backbone"] + t["encdec"] + t["postprocess"] - t["total"]) < 0.05 * t["total"] + 0.05
    assert det.detect(img) == det.detect(img)
