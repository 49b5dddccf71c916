"""Precision-mode variants on the tensor cores (reference
tensors.py:111-170, pipeline.py:318-367): the fp16-storage discipline and the fp16-accumulate
negative control of the tcgen05 GEMM (dart_gemm_force_precision / dart_model_set_precision),
and `precision_study` against the reference's own study (tests/golden/golden_S.npz,
oracle/make_golden.py S)."""

import json
import math
import os

import numpy as np
import pytest

from conftest import load_golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2603_11441_b200 as D  # noqa: E402
from paper_2603_11441_b200 import _native  # noqa: E402
from paper_2603_11441_b200.model import native_handle  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return _native.load()


def gemm(lib, A, W, bias, epi, out, precision):
    M, K = A.shape
    lib.dart_gemm_force_precision(precision)
    try:
        _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None, M, W.shape[0],
                                    K, epi, None, None, 0, 0, 0, torch.cuda.current_stream().cuda_stream))
    finally:
        lib.dart_gemm_force_precision(0)
    torch.cuda.synchronize()
    return out


def f16_storage(x):
    """The reference's half_round: saturate at +-65504, round to binary16 (tensors.py:99-109)."""
    return x.clamp(-65504.0, 65504.0).half().float()


@pytest.mark.parametrize("M,N,K", [(300, 192, 128), (5184, 1280, 5120)])
def test_fp16_storage_rounds_fp32_outputs(lib, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M + N)
    A = torch.randn(M, K, device="cuda", generator=g).half()
    W = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).half()
    bias = torch.randn(N, device="cuda", generator=g)
    o0 = gemm(lib, A, W, bias, 2, torch.empty(M, N, device="cuda"), 0)
    o1 = gemm(lib, A, W, bias, 2, torch.empty(M, N, device="cuda"), 1)
    assert torch.equal(o1, f16_storage(o0))
    # residual stream: x <- half(x + acc + b)
    x0 = torch.randn(M, N, device="cuda", generator=g) * 100
    r0 = gemm(lib, A, W, bias, 3, x0.clone(), 0)
    r1 = gemm(lib, A, W, bias, 3, x0.clone(), 1)
    assert torch.equal(r1, f16_storage(r0))


@pytest.mark.parametrize("M,N,K", [(1000, 256, 1280), (5184, 1280, 5120)])
def test_fp16_accumulation_is_the_lossy_control(lib, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(K)
    A = torch.randn(M, K, device="cuda", generator=g).half()
    W = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).half()
    bias = torch.zeros(N, device="cuda")
    ref = A.float() @ W.float().T
    o1 = gemm(lib, A, W, bias, 2, torch.empty(M, N, device="cuda"), 1)
    o2 = gemm(lib, A, W, bias, 2, torch.empty(M, N, device="cuda"), 2)
    assert torch.equal(o2, o2.half().float())  # fp16 values
    e1 = (o1 - ref).abs().mean().item()
    e2 = (o2 - ref).abs().mean().item()
    # fp16 partial sums lose bits on every accumulate step: strictly worse than fp16 storage
    # of an fp32-accumulated result, but still the same GEMM (not garbage)
    assert e2 > 1.5 * e1, (e1, e2)
    assert float((o2 - ref).abs().max() / ref.abs().max()) < 3e-2


def test_fp16_accumulator_overflows(lib):
    """+64 x 1536 then -64 x 1536: the exact sum is 0, but the running fp16 sum passes 65504."""
    M, N, K = 256, 256, 3072
    A = torch.full((M, K), 64.0, device="cuda")
    A[:, K // 2:] = -64.0
    A = A.half()
    W = torch.ones(N, K, device="cuda").half()
    bias = torch.zeros(N, device="cuda")
    o1 = gemm(lib, A, W, bias, 2, torch.empty(M, N, device="cuda"), 1)
    o2 = gemm(lib, A, W, bias, 2, torch.empty(M, N, device="cuda"), 2)
    assert torch.count_nonzero(o1).item() == 0
    assert o2.abs().min().item() >= 1024.0  # the overflowed accumulator never comes back


def _study_setup():
    g = load_golden("S")
    cfg = D.ModelConfig.from_dict(json.loads(str(g["config_json"])))
    model = D.build_model(cfg, with_mask_head=False)
    assert D.weights_checksum(model) == str(g["weights_checksum"])
    images = [D.generate_scene(D.SceneSpec(seed=int(s), num_classes=3))[0] for s in g["seeds"]]
    return g, model, images


def test_precision_study_matches_reference_ordering():
    g, model, images = _study_setup()
    depths = [int(d) for d in g["depths"]]
    # the full-precision side of the study is within 1e-4 of the reference's float64 features
    for i, d in enumerate(depths):
        tm = D.truncate_model(model, d)
        for j, img in enumerate(images):
            l0 = D.backbone_forward(tm, img).levels[0]
            assert D.cosine_similarity(l0, g["l0_fp32"][i, j]) > 0.9999
    rep = D.precision_study(model, images, depths)
    ref_rows = {(int(d), str(m)): v for (d, v), m in zip(g["cosines"], g["modes"])}
    assert [(d, m) for d, m, _ in rep.rows] == [(int(d), str(m)) for (d, _), m in zip(g["cosines"], g["modes"])]
    for d in depths:
        c32 = rep.cosine(d, D.PrecisionMode.FP16_ACCUM_FP32)
        c16 = rep.cosine(d, D.PrecisionMode.FP16_ACCUM_FP16)
        assert c32 > 0.9999 and c16 > 0.999
        # the reference's ordering: fp16 accumulation degrades more than fp16 storage
        assert ref_rows[(d, "fp16-accum-fp16")] < ref_rows[(d, "fp16-accum-fp32")]
        assert c16 < c32, (d, c16, c32)
    # the study leaves the handle on the detection discipline
    h = native_handle(D.truncate_model(model, depths[-1]))
    assert h.lib.dart_model_get_precision(h.ptr) == 0


def test_precision_study_full_vit_h():
    """Table 6 analogue at full size (ViT-H/14, 1008^2): fp16 storage stays correct through 32
    blocks; fp16 accumulation is the degraded control.  Writes the table to gpurun_out/."""
    model = D.build_model(D.vit_h_config(), with_mask_head=False)
    images = [D.generate_scene(D.SceneSpec(seed=100 + i, image_size=1008, num_classes=4))[0] for i in range(5)]
    depths = [8, 16, 32]
    rep = D.precision_study(model, images, depths)
    os.makedirs("gpurun_out", exist_ok=True)
    with open(os.path.join("gpurun_out", "precision_study_vit_h.json"), "w") as f:
        json.dump(rep.to_table(), f, indent=1)
    for d in depths:
        assert rep.cosine(d, D.PrecisionMode.FP16_ACCUM_FP32) > 0.999
    assert rep.cosine(32, D.PrecisionMode.FP16_ACCUM_FP16) < rep.cosine(32, D.PrecisionMode.FP16_ACCUM_FP32)
