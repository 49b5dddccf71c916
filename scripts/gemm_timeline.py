"""Per-CTA timeline of one persistent GEMM launch (dart_gemm_trace globaltimer stamps) at the DART
backbone shapes, launched right after a warm-up launch of the same GEMM (as in a step).
    python scripts/gemm_timeline.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()
names = ["entry", "pdl_ok", "1st data", "1st commit", "epi sees 1st", "epi done", "last commit", "exit"]
for label, M, N, K, epi in (("attn.out", 5184, 1280, 1280, 3), ("mlp.fc2", 5184, 1280, 5120, 3),
                            ("mlp.fc1", 5184, 5120, 1280, 1), ("1 tile/pair", 256 * 37, 1280, 1280, 3)):
    A = torch.randn(M, K, device="cuda").half()
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).half()
    bias = torch.zeros(N, device="cuda")
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 3 else torch.float16)
    tr = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    f = lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None, M, N, K,
                                            epi, None, None, 0, 0, 0, st.cuda_stream))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    f()  # predecessor
    _native.check(lib.dart_gemm_trace(tr.data_ptr()))
    f()
    _native.check(lib.dart_gemm_trace(None))
    f()
    torch.cuda.synchronize()
    t = tr.cpu().numpy().reshape(148, 8).astype(np.float64)
    used = t[:, 0] > 0
    t = t[used]
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0  # us
    rel[t == 0] = np.nan
    print(f"== {label} M={M} N={N} K={K} epi {epi}: {used.sum()} CTAs, kernel span {np.nanmax(rel[:, 7]):.2f} us")
    for i, n in enumerate(names):
        col = rel[:, i]
        if np.all(np.isnan(col)):
            continue
        print(f"   {n:13s} min {np.nanmin(col):7.2f}  median {np.nanmedian(col):7.2f}  max {np.nanmax(col):7.2f} us")
