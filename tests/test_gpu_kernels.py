"""Per-kernel numerics on the B200: the tcgen05 GEMM (every epilogue) and the flash
attention, each against a plain PyTorch fp32 reference of the same op, called through
the C ABI (dart_gemm / dart_attention)."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2603_11441_b200 import _native  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.backends.cuda.matmul.allow_tf32 = False
    return _native.load()


def stream():
    return torch.cuda.current_stream().cuda_stream


def run_gemm(lib, A, W, bias, epi, out, out2=None, rope=None):
    M, K = A.shape
    N = W.shape[0]
    rc, rs, rT, rhd, rcols = (None, None, 0, 0, 0) if rope is None else rope
    _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr() if bias is not None else None,
                                out.data_ptr(), out2.data_ptr() if out2 is not None else None, M, N, K, epi,
                                rc.data_ptr() if rc is not None else None, rs.data_ptr() if rs is not None else None,
                                rT, rhd, rcols, stream()))
    torch.cuda.synchronize()


def rel_err(got, ref):
    return float((got.float() - ref).abs().max() / ref.abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (300, 192, 128), (1000, 256, 1280), (5184, 3840, 1280),
                                   (5184, 1280, 5120), (777, 512, 256), (201, 1024, 256), (64, 3072, 256)])
def test_gemm_f32_out(lib, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A = torch.randn(M, K, device="cuda", generator=g).half()
    W = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).half()
    bias = torch.randn(N, device="cuda", generator=g)
    out = torch.empty(M, N, device="cuda")
    run_gemm(lib, A, W, bias, 2, out)
    ref = A.float() @ W.float().T + bias
    assert rel_err(out, ref) < 1e-5


@pytest.mark.parametrize("epi", [0, 1, 3, 5])
def test_gemm_epilogues(lib, epi):
    M, N, K = 517, 768, 320
    g = torch.Generator(device="cuda").manual_seed(epi)
    A = torch.randn(M, K, device="cuda", generator=g).half()
    W = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).half()
    bias = torch.randn(N, device="cuda", generator=g)
    ref = A.float() @ W.float().T + bias
    if epi in (0, 1):
        out = torch.empty(M, N, device="cuda", dtype=torch.float16)
        run_gemm(lib, A, W, bias, epi, out)
        if epi == 1:
            ref = ref.clamp_min(0)
        assert rel_err(out, ref) < 2e-3
    elif epi == 3:
        resid = torch.randn(M, N, device="cuda", generator=g)
        out = resid.clone()
        run_gemm(lib, A, W, bias, 3, out)
        assert rel_err(out, ref + resid) < 1e-5
    else:
        out = torch.empty(M, N, device="cuda")
        out2 = torch.empty(M, N, device="cuda", dtype=torch.float16)
        run_gemm(lib, A, W, bias, 5, out, out2)
        assert rel_err(out, ref) < 1e-5 and rel_err(out2, ref) < 2e-3


PLANS = [(256, 1), (128, 1), (64, 1), (256, 2), (192, 2), (160, 2), (128, 2), (64, 2)]


@pytest.mark.parametrize("bn,cg", [(256, 2), (128, 2), (256, 1), (128, 1)])
@pytest.mark.parametrize("M,N,K", [(5184, 1280, 5120), (5184, 1280, 1280), (1333, 768, 640), (300, 256, 128)])
def test_gemm_split_k_residual(lib, bn, cg, M, N, K):
    """Split-K residual epilogue: every tile as two K halves; the half that reaches its epilogue
    second adds the first's partial accumulator and does out += bias + acc.  Equal to fp32 torch,
    deterministic, and bitwise independent of M (rows computed inside a larger launch -- other
    tiles, other claim orders -- are the same bits)."""
    g = torch.Generator(device="cuda").manual_seed(M + N + K + bn)
    A = torch.randn(2 * M, K, device="cuda", generator=g).half()
    W = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).half()
    bias = torch.randn(N, device="cuda", generator=g)
    x0 = torch.randn(2 * M, N, device="cuda", generator=g)
    ref = x0[:M] + A[:M].float() @ W.float().T + bias
    outs = []
    lib.dart_gemm_force_plan(bn, cg)
    lib.dart_gemm_force_splitk(2)
    try:
        for rows in (M, M, 2 * M):
            out = x0[:rows].clone()
            _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None, rows, N, K,
                                        3, None, None, 0, 0, 0, stream()))
            outs.append(out[:M])
        torch.cuda.synchronize()
    finally:
        lib.dart_gemm_force_splitk(1)
        lib.dart_gemm_force_plan(0, 0)
    assert rel_err(outs[0], ref) < 2e-5
    assert torch.equal(outs[0], outs[1])
    assert torch.equal(outs[0], outs[2])


@pytest.mark.parametrize("epi", [0, 1, 2, 4, 5])
def test_gemm_split_k_epilogues(lib, epi):
    """Split-K through every other epilogue (bias / ReLU / RoPE after the two halves combine), on the
    backbone's QKV shape (315 CTA-pair tiles) and a ragged one; rows bitwise independent of M."""
    T, E = 5184, 1280
    M, N, K = (5184, 3840, 1280) if epi == 4 else (1700, 768, 640)
    g = torch.Generator(device="cuda").manual_seed(epi + 11)
    A = torch.randn(M + 700, K, device="cuda", generator=g).half()
    W = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).half()
    bias = torch.randn(N, device="cuda", generator=g)
    ref = A[:M].float() @ W.float().T + bias
    f16 = epi in (0, 1, 4)
    rope = None
    if epi == 4:
        hd, H = 80, 16
        cos, sin = rope_tables(72, hd)
        rope = (cos, sin, T, hd, 2 * E)
        y = ref.reshape(M, 3, H, hd)
        tok = torch.arange(M, device="cuda") % T
        c, s = cos[tok][:, None, None, :], sin[tok][:, None, None, :]
        rot = y.clone()
        rot[:, :2, :, 0::2] = (y[..., 0::2] * c - y[..., 1::2] * s)[:, :2]
        rot[:, :2, :, 1::2] = (y[..., 0::2] * s + y[..., 1::2] * c)[:, :2]
        ref = rot.reshape(M, N)
    elif epi == 1:
        ref = ref.clamp_min(0)
    outs = []
    lib.dart_gemm_force_splitk(2)
    try:
        for rows in (M, M + 700):
            out = torch.empty(rows, N, device="cuda", dtype=torch.float16 if f16 else torch.float32)
            out2 = torch.empty(rows, N, device="cuda", dtype=torch.float16) if epi == 5 else None
            run_gemm(lib, A[:rows], W, bias, epi, out, out2, rope=rope)
            outs.append((out[:M], out2[:M] if out2 is not None else None))
    finally:
        lib.dart_gemm_force_splitk(1)
    assert rel_err(outs[0][0], ref) < (2e-3 if f16 else 2e-5)
    assert torch.equal(outs[0][0], outs[1][0])
    if epi == 5:
        assert rel_err(outs[0][1], ref) < 2e-3 and torch.equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("bn,cg", PLANS)
@pytest.mark.parametrize("epi", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("shape", ["waves", "tail"])
def test_gemm_forced_plans(lib, bn, cg, epi, shape):
    """Every tile plan (1-SM 128 x bn and CTA-pair 256 x bn tiles) and epilogue, with M and N tails
    that leave partial 256-row tiles and several waves.  "tail": the DART shapes whose last wave
    is at most half full (5184 x 1280: 105 CTA-pair tiles; 5184 x 3840: 315), which run that wave
    as half-width units."""
    T, E = 576, 1280
    if shape == "tail":
        M, N, K = (5184, 3840, 1280) if epi == 4 else (5184, 1280, 640)
        if N % bn:
            pytest.skip("bn does not divide N")
    else:
        M, N, K = (1700, 3840, 1280) if epi == 4 else (5000, 6 * bn, 320)
    g = torch.Generator(device="cuda").manual_seed(bn * 10 + cg + epi)
    A = torch.randn(M, K, device="cuda", generator=g).half()
    W = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).half()
    bias = torch.randn(N, device="cuda", generator=g)
    ref = A.float() @ W.float().T + bias
    lib.dart_gemm_force_plan(bn, cg)
    try:
        if epi in (0, 1):
            out = torch.empty(M, N, device="cuda", dtype=torch.float16)
            run_gemm(lib, A, W, bias, epi, out)
            assert rel_err(out, ref.clamp_min(0) if epi == 1 else ref) < 2e-3
        elif epi == 2:
            out = torch.empty(M, N, device="cuda")
            run_gemm(lib, A, W, bias, 2, out)
            assert rel_err(out, ref) < 1e-5
        elif epi == 3:
            resid = torch.randn(M, N, device="cuda", generator=g)
            out = resid.clone()
            run_gemm(lib, A, W, bias, 3, out)
            assert rel_err(out, ref + resid) < 1e-5
        elif epi == 4:
            hd, H = 80, 16
            cos, sin = rope_tables(24, hd)
            out = torch.empty(M, N, device="cuda", dtype=torch.float16)
            run_gemm(lib, A, W, bias, 4, out, rope=(cos, sin, T, hd, 2 * E))
            y = ref.reshape(M, 3, H, hd)
            tok = torch.arange(M, device="cuda") % T
            c, s = cos[tok][:, None, None, :], sin[tok][:, None, None, :]
            rot = y.clone()
            rot[:, :2, :, 0::2] = (y[..., 0::2] * c - y[..., 1::2] * s)[:, :2]
            rot[:, :2, :, 1::2] = (y[..., 0::2] * s + y[..., 1::2] * c)[:, :2]
            assert rel_err(out, rot.reshape(M, N)) < 2e-3
        else:
            out = torch.empty(M, N, device="cuda")
            out2 = torch.empty(M, N, device="cuda", dtype=torch.float16)
            run_gemm(lib, A, W, bias, 5, out, out2)
            assert rel_err(out, ref) < 1e-5 and rel_err(out2, ref) < 2e-3
    finally:
        lib.dart_gemm_force_plan(0, 0)


def rope_tables(grid, hd):
    """The reference's 2-D RoPE tables (model.py:203-213): [T, hd/2] = [row angles | col angles]."""
    q = hd // 4
    inv = 100.0 ** (-torch.arange(q, dtype=torch.float64) / q)
    r = torch.arange(grid, dtype=torch.float64).repeat_interleave(grid)
    c = torch.arange(grid, dtype=torch.float64).repeat(grid)
    ang = torch.cat([r[:, None] * inv, c[:, None] * inv], 1)
    return torch.cos(ang).float().cuda().contiguous(), torch.sin(ang).float().cuda().contiguous()


@pytest.mark.parametrize("T,M", [(576, 576), (5184, 5184), (576, 1152)])
def test_gemm_rope_epilogue(lib, T, M):
    """QKV projection with RoPE on q and k (reference model.py:392-397, tensors.py:235-252)."""
    E, H = 1280, 16
    hd = E // H
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(M, E, device="cuda", generator=g).half()
    W = (torch.randn(3 * E, E, device="cuda", generator=g) / math.sqrt(E)).half()
    bias = torch.randn(3 * E, device="cuda", generator=g)
    cos, sin = rope_tables(int(round(T ** 0.5)), hd)
    out = torch.empty(M, 3 * E, device="cuda", dtype=torch.float16)
    run_gemm(lib, A, W, bias, 4, out, rope=(cos, sin, T, hd, 2 * E))
    y = (A.float() @ W.float().T + bias).reshape(M, 3, H, hd)
    ev, od = y[..., 0::2], y[..., 1::2]
    tok = torch.arange(M, device="cuda") % T
    c, s = cos[tok][:, None, None, :], sin[tok][:, None, None, :]
    rot = torch.empty_like(y)
    rot[..., 0::2] = ev * c - od * s
    rot[..., 1::2] = ev * s + od * c
    rot[:, 2] = y[:, 2]
    assert rel_err(out, rot.reshape(M, 3 * E)) < 2e-3


def ref_attention(q, k, v):
    s = (q.float() @ k.float().transpose(-1, -2)) / math.sqrt(q.shape[-1])
    return torch.softmax(s, dim=-1) @ v.float()


@pytest.mark.parametrize("hd,Lq,Lk,heads,batch", [(80, 576, 576, 16, 2), (80, 5184, 5184, 2, 1), (16, 5184, 5184, 4, 2),
                                                  (16, 5184, 32, 16, 13), (16, 4000, 20, 16, 17),
                                                  (16, 201, 5184, 16, 3), (16, 5184, 32, 16, 2), (16, 201, 201, 16, 2),
                                                  (16, 64, 64, 4, 1), (16, 17, 8, 4, 1)])
def test_attention_dense(lib, hd, Lq, Lk, heads, batch):
    g = torch.Generator(device="cuda").manual_seed(hd + Lq + Lk)
    q = (torch.randn(batch, Lq, heads, hd, device="cuda", generator=g) * 2).half()
    k = (torch.randn(batch, Lk, heads, hd, device="cuda", generator=g) * 2).half()
    v = torch.randn(batch, Lk, heads, hd, device="cuda", generator=g).half()
    o = torch.empty(batch, Lq, heads, hd, device="cuda", dtype=torch.float16)
    _native.check(lib.dart_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), batch, heads, Lq, Lk,
                                     hd, heads * hd, heads * hd, heads * hd, Lq * heads * hd, Lk * heads * hd,
                                     Lq * heads * hd, 0, 0, stream()))
    torch.cuda.synchronize()
    ref = ref_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2)).transpose(1, 2)
    assert float((o.float() - ref).abs().max()) < 1e-2


@pytest.mark.parametrize("hd,grid,win,heads", [(80, 72, 24, 16), (16, 8, 4, 4)])
def test_attention_windowed(lib, hd, grid, win, heads):
    """Windowed attention reads the token-major QKV directly (model.py:375-387, 398-408)."""
    T = grid * grid
    B = 2
    g = torch.Generator(device="cuda").manual_seed(hd)
    qkv = (torch.randn(B, T, 3, heads, hd, device="cuda", generator=g) * 2).half()
    o = torch.empty(B, T, heads * hd, device="cuda", dtype=torch.float16)
    E = heads * hd
    base = qkv.reshape(B, T, 3 * E)
    nw = (grid // win) ** 2
    _native.check(lib.dart_attention(base.data_ptr(), base[..., E:].data_ptr(), base[..., 2 * E:].data_ptr(),
                                     o.data_ptr(), B * nw, heads, win * win, win * win, hd, 3 * E, 3 * E, E,
                                     T * 3 * E, T * 3 * E, T * E, win, grid, stream()))
    torch.cuda.synchronize()
    n = grid // win
    x = qkv.reshape(B, n, win, n, win, 3, heads, hd).permute(0, 1, 3, 5, 6, 2, 4, 7).reshape(B, n * n, 3, heads, win * win, hd)
    ow = ref_attention(x[:, :, 0], x[:, :, 1], x[:, :, 2])  # [B, nw, H, w2, hd]
    ow = ow.reshape(B, n, n, heads, win, win, hd).permute(0, 1, 4, 2, 5, 3, 6).reshape(B, T, E)
    assert float((o.float() - ow).abs().max()) < 1e-2


@pytest.mark.parametrize("items,L,hd", [(2, 576, 80), (1, 5184, 80), (9, 576, 80), (2, 5184, 16), (3, 576, 16)])
def test_attention_tcgen05_packed_qkv(lib, items, L, hd):
    """tcgen05/TMEM flash attention (hd 80 backbone, hd 16 enc-dec) on a packed QKV layout vs fp32 torch."""
    H = 16
    E = H * hd
    g = torch.Generator(device="cuda").manual_seed(L + items)
    qkv = (torch.randn(items, L, 3, H, hd, device="cuda", generator=g) * 2).half()
    o = torch.empty(items, L, E, device="cuda", dtype=torch.float16)
    _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o.data_ptr(), items, H, L, hd, None, stream()))
    torch.cuda.synchronize()
    x = qkv.permute(2, 0, 3, 1, 4)  # [3, items, H, L, hd]
    ref = ref_attention(x[0], x[1], x[2]).permute(0, 2, 1, 3).reshape(items, L, E)
    assert float((o.float() - ref).abs().max()) < 1e-2


@pytest.mark.parametrize("M,K", [(300, 256), (20736, 256), (804, 1024), (5184 * 3, 256)])
def test_gemm_residual_layernorm_epilogue(lib, M, K):
    """EPI_F32_RESID_LN: x += A W^T + b and h = LN(x) g + beta in the same epilogue (the enc-dec's
    fused sub-block boundary) vs fp32 torch; x also equals the plain residual GEMM's x bitwise."""
    g = torch.Generator(device="cuda").manual_seed(M + K)
    A = torch.randn(M, K, device="cuda", generator=g).half()
    W = (torch.randn(256, K, device="cuda", generator=g) / math.sqrt(K)).half()
    bias = torch.randn(256, device="cuda", generator=g) * 0.1
    x0 = torch.randn(M, 256, device="cuda", generator=g) * 3 + 1.5  # offset rows: the mean matters
    gam = torch.rand(256, device="cuda", generator=g) + 0.5
    bet = torch.randn(256, device="cuda", generator=g) * 0.2
    x = x0.clone()
    h = torch.empty(M, 256, device="cuda", dtype=torch.float16)
    _native.check(lib.dart_gemm_resid_ln(A.data_ptr(), W.data_ptr(), bias.data_ptr(), x.data_ptr(), h.data_ptr(),
                                         gam.data_ptr(), bet.data_ptr(), M, K, stream()))
    x_plain = x0.clone()
    run_gemm(lib, A, W, bias, 3, x_plain)
    torch.cuda.synchronize()
    assert torch.equal(x, x_plain)
    ref_x = x0 + A.float() @ W.float().t() + bias
    assert rel_err(x, ref_x) < 2e-3
    ref_h = torch.nn.functional.layer_norm(x, (256,), gam, bet, eps=1e-6)
    assert float((h.float() - ref_h).abs().max()) < 2e-2


@pytest.mark.parametrize("items,L,hd", [(3, 201, 16), (5, 16, 16), (2, 32, 16), (7, 20, 16), (4, 64, 16),
                                        (2, 100, 80), (1, 201, 80)])
def test_attention_tcgen05_ragged_keys(lib, items, L, hd):
    """Key counts that are not a multiple of the key tile run the masked tcgen05 kernel (keys past L
    in the last tile get P = 0): the decoder's 201-token self-attention (model.py:525), the short
    32-key tile path (text cross-attention, model.py:518) and toy-size windows, vs fp32 torch."""
    H = 16
    E = H * hd
    g = torch.Generator(device="cuda").manual_seed(L * 7 + items)
    qkv = (torch.randn(items, L, 3, H, hd, device="cuda", generator=g) * 2).half()
    o = torch.full((items, L, E), float("nan"), device="cuda", dtype=torch.float16)
    _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o.data_ptr(), items, H, L, hd, None, stream()))
    torch.cuda.synchronize()
    x = qkv.permute(2, 0, 3, 1, 4)
    ref = ref_attention(x[0], x[1], x[2]).permute(0, 2, 1, 3).reshape(items, L, E)
    assert bool(torch.isfinite(o).all())
    assert float((o.float() - ref).abs().max()) < 1e-2


@pytest.mark.parametrize("hd,L", [(80, 576), (16, 576), (80, 5184)])
@pytest.mark.parametrize("mixed", [False, True])
def test_attention_tcgen05_large_logits(lib, hd, L, mixed):
    """Peaked softmax: scores growing along the key axis overflow the fixed-reference pass (first
    key tile's max), so those items are recomputed by the max-tracking pass.  mixed: only half of
    the heads overflow (per-item selection of the second pass)."""
    items, H = 1, 16
    E = H * hd
    g = torch.Generator(device="cuda").manual_seed(7)
    qkv = torch.randn(items, L, 3, H, hd, device="cuda", generator=g)
    qkv[:, :, 0] *= 4
    grow = torch.linspace(0.1, 6 if hd == 80 else 14, L, device="cuda")[None, :, None, None]
    if mixed:
        qkv[:, :, 1, : H // 2] *= grow
    else:
        qkv[:, :, 1] *= grow
    qkv = qkv.half()
    o = torch.empty(items, L, E, device="cuda", dtype=torch.float16)
    _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o.data_ptr(), items, H, L, hd, None, stream()))
    torch.cuda.synchronize()
    x = qkv.permute(2, 0, 3, 1, 4)
    ref = ref_attention(x[0], x[1], x[2]).permute(0, 2, 1, 3).reshape(items, L, E)
    assert float((o.float() - ref).abs().max()) < 2e-2


@pytest.mark.parametrize("items,L,hd", [(2, 576, 80), (2, 5184, 16)])
def test_attention_tcgen05_forced_safe_pass(lib, items, L, hd):
    """Every item re-run through the max-tracking pass gives the same result as the fast pass."""
    H = 16
    E = H * hd
    g = torch.Generator(device="cuda").manual_seed(L + items)
    qkv = (torch.randn(items, L, 3, H, hd, device="cuda", generator=g) * 2).half()
    o1 = torch.empty(items, L, E, device="cuda", dtype=torch.float16)
    o2 = torch.empty_like(o1)
    _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o1.data_ptr(), items, H, L, hd, None, stream()))
    lib.dart_attention_force_safe(1)
    try:
        _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o2.data_ptr(), items, H, L, hd, None, stream()))
    finally:
        lib.dart_attention_force_safe(0)
    torch.cuda.synchronize()
    x = qkv.permute(2, 0, 3, 1, 4)
    ref = ref_attention(x[0], x[1], x[2]).permute(0, 2, 1, 3).reshape(items, L, E)
    assert float((o1.float() - ref).abs().max()) < 1e-2
    assert float((o2.float() - ref).abs().max()) < 1e-2


@pytest.mark.parametrize("items,L,hd", [(1, 5184, 80), (9, 576, 80), (3, 5184, 16)])
def test_attention_tcgen05_production_equals_hooked(lib, items, L, hd):
    """The default launch runs the hook-free production instantiation; with a trace buffer set
    it runs the hooked twin.  Same arithmetic: outputs bitwise equal."""
    H = 16
    E = H * hd
    g = torch.Generator(device="cuda").manual_seed(7 * L + items)
    qkv = torch.randn(items * L, 3 * E, device="cuda", generator=g).half()
    o1 = torch.empty(items * L, E, device="cuda", dtype=torch.float16)
    o2 = torch.empty_like(o1)
    tr = torch.zeros(11 * 256, dtype=torch.int64, device="cuda")
    _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o1.data_ptr(), items, H, L, hd, None, stream()))
    lib.dart_attention_trace(tr.data_ptr())
    try:
        _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o2.data_ptr(), items, H, L, hd, None, stream()))
        torch.cuda.synchronize()
    finally:
        lib.dart_attention_trace(None)
    assert torch.equal(o1, o2)
    assert int(tr.count_nonzero()) > 0  # the hooked twin really ran (it wrote its stamps)


@pytest.mark.parametrize("rows,dim,f16", [(5184, 1280, 1), (20736, 256, 1), (777, 256, 0), (1001, 1280, 1), (33, 64, 1)])
def test_layernorm(lib, rows, dim, f16):
    """LayerNorm (population variance, eps 1e-6; reference tensors.py:215-227) vs fp32 torch."""
    g = torch.Generator(device="cuda").manual_seed(rows + dim)
    x = torch.randn(rows, dim, device="cuda", generator=g) * 3 + 1.5
    gamma = torch.randn(dim, device="cuda", generator=g)
    beta = torch.randn(dim, device="cuda", generator=g)
    y = torch.empty(rows, dim, device="cuda", dtype=torch.float16 if f16 else torch.float32)
    _native.check(lib.dart_layernorm(x.data_ptr(), gamma.data_ptr(), beta.data_ptr(), y.data_ptr(), rows, dim, f16,
                                     stream()))
    torch.cuda.synchronize()
    ref = torch.nn.functional.layer_norm(x, (dim,), gamma, beta, eps=1e-6)
    assert float((y.float() - ref).abs().max()) < (1e-2 if f16 else 1e-4)


@pytest.mark.parametrize("M", [300, 5184, 20736, 41472 + 77])
def test_mlp_fused(lib, M):
    """Fused enc-dec MLP (hidden activations in TMEM): x += relu(h W1^T + b1) W2^T + b2 vs fp32 torch
    with the same fp16 rounding of h, the weights and the hidden activations."""
    g = torch.Generator(device="cuda").manual_seed(M)
    h = torch.randn(M, 256, device="cuda", generator=g).half()
    w1 = (torch.randn(1024, 256, device="cuda", generator=g) / 16).half()
    w2 = (torch.randn(256, 1024, device="cuda", generator=g) / 32).half()
    b1 = torch.randn(1024, device="cuda", generator=g) * 0.1
    b2 = torch.randn(256, device="cuda", generator=g) * 0.1
    x = torch.randn(M, 256, device="cuda", generator=g)
    hid = torch.relu(h.float() @ w1.float().T + b1).half().float()
    ref = x + hid @ w2.float().T + b2
    out = x.clone()
    _native.check(lib.dart_mlp_fused(h.data_ptr(), w1.data_ptr(), b1.data_ptr(), w2.data_ptr(), b2.data_ptr(),
                                     out.data_ptr(), M, stream()))
    torch.cuda.synchronize()
    assert rel_err(out, ref) < 2e-3


@pytest.mark.parametrize("M", [300, 20736, 41472, 75776 + 77])  # last: several units per CTA pair, ragged tail
def test_mlp_fused_layernorm_equals_gemm_path(lib, M):
    """The fused MLP kernel's LN epilogue and the GEMM path (fc1 GEMM + fc2 GEMM with the
    EPI_F32_RESID_LN epilogue) give identical bits for x and h = LN(x): the enc-dec picks one or
    the other by row count (i.e. by class count), and a class's outputs must not depend on N."""
    g = torch.Generator(device="cuda").manual_seed(M + 1)
    h = torch.randn(M, 256, device="cuda", generator=g).half()
    w1 = (torch.randn(1024, 256, device="cuda", generator=g) / 16).half()
    w2 = (torch.randn(256, 1024, device="cuda", generator=g) / 32).half()
    b1 = torch.randn(1024, device="cuda", generator=g) * 0.1
    b2 = torch.randn(256, device="cuda", generator=g) * 0.1
    x0 = torch.randn(M, 256, device="cuda", generator=g) * 2 + 0.7
    gam = torch.rand(256, device="cuda", generator=g) + 0.5
    bet = torch.randn(256, device="cuda", generator=g) * 0.2
    x_f, h_f = x0.clone(), h.clone()  # fused kernel, LN written over its own input (as the enc-dec does)
    _native.check(lib.dart_mlp_fused_ln(h_f.data_ptr(), w1.data_ptr(), b1.data_ptr(), w2.data_ptr(), b2.data_ptr(),
                                        x_f.data_ptr(), h_f.data_ptr(), gam.data_ptr(), bet.data_ptr(), M, stream()))
    hid = torch.empty(M, 1024, device="cuda", dtype=torch.float16)
    run_gemm(lib, h, w1, b1, 1, hid)
    x_g, h_g = x0.clone(), torch.empty(M, 256, device="cuda", dtype=torch.float16)
    _native.check(lib.dart_gemm_resid_ln(hid.data_ptr(), w2.data_ptr(), b2.data_ptr(), x_g.data_ptr(), h_g.data_ptr(),
                                         gam.data_ptr(), bet.data_ptr(), M, 1024, stream()))
    torch.cuda.synchronize()
    assert torch.equal(x_f, x_g)
    assert torch.equal(h_f, h_g)
    ref = torch.nn.functional.layer_norm(x_g, (256,), gam, bet, eps=1e-6)
    assert float((h_g.float() - ref).abs().max()) < 2e-2
