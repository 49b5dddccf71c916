"""Per-unit timeline (dart_gemm_trace) of the backbone QKV GEMM with and without the RoPE epilogue
(M = 5184, N = 3840, K = 1280).  python scripts/gemm_qkv_timeline.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()
M, N, K, T, hd = 5184, 3840, 1280, 5184, 80
A = torch.randn(M, K, device="cuda").half()
W = (torch.randn(N, K, device="cuda") / K ** 0.5).half()
bias = torch.zeros(N, device="cuda")
out = torch.empty(M, N, device="cuda", dtype=torch.float16)
q = hd // 4
inv = 100.0 ** (-torch.arange(q, dtype=torch.float64) / q)
r = torch.arange(72, dtype=torch.float64).repeat_interleave(72)
c = torch.arange(72, dtype=torch.float64).repeat(72)
ang = torch.cat([r[:, None] * inv, c[:, None] * inv], 1)
cos, sin = torch.cos(ang).float().cuda().contiguous(), torch.sin(ang).float().cuda().contiguous()
for epi in (0, 4):
    def f():
        _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None, M, N, K, epi,
                                    cos.data_ptr() if epi == 4 else None, sin.data_ptr() if epi == 4 else None,
                                    T if epi == 4 else 0, hd if epi == 4 else 0, 2 * 1280 if epi == 4 else 0,
                                    st.cuda_stream))
    tr = torch.zeros(148 * 8 + 148 * 64, dtype=torch.int64, device="cuda")
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    f()
    _native.check(lib.dart_gemm_trace(tr.data_ptr()))
    f()
    _native.check(lib.dart_gemm_trace(None))
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.float64)
    cta = t[:148 * 8].reshape(148, 8)
    u = t[148 * 8:].reshape(148, 8, 8)
    t0 = cta[cta[:, 0] > 0, 0].min()
    print(f"== epi {epi}: {e0.elapsed_time(e1) / 20 * 1000:.1f} us per launch, traced span {(cta[:, 7].max() - t0) / 1e3:.2f} us")
    for k in (0, 1, 40, 100):
        row = []
        for it in range(8):
            if u[k, it, 1] == 0:
                continue
            row.append(f"u{it}[mma {(u[k, it, 0] - t0) / 1e3:.1f} acc {(u[k, it, 1] - t0) / 1e3:.1f} epi {(u[k, it, 6] - t0) / 1e3:.1f}]")
        print(f"  cta {k:3d}: " + "  ".join(row))
