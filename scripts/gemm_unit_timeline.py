"""Per-unit timeline (dart_gemm_trace per-unit stamps, warp 4 of each CTA) of one persistent GEMM
launch, with and without split-K.  python scripts/gemm_unit_timeline.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()
ev = ["mma issued", "acc ready", "part stored", "published", "comb wait0", "part visible", "epi done"]
SPLITS = [int(a) for a in sys.argv[1:]] or [1, 2]
for label, M, N, K, epi in (("attn.out", 5184, 1280, 1280, 3), ("mlp.fc2", 5184, 1280, 5120, 3),
                            ("mlp.fc1", 5184, 5120, 1280, 1), ("epi-only K=64", 5184 * 4, 1280, 64, 0)):
    A = torch.randn(M, K, device="cuda").half()
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).half()
    bias = torch.zeros(N, device="cuda")
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 3 else torch.float16)
    for sk in SPLITS:
        lib.dart_gemm_force_splitk(sk)
        tr = torch.zeros(148 * 8 + 148 * 64, dtype=torch.int64, device="cuda")
        f = lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None, M, N,
                                                K, epi, None, None, 0, 0, 0, st.cuda_stream))
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        f()
        _native.check(lib.dart_gemm_trace(tr.data_ptr()))
        f()
        _native.check(lib.dart_gemm_trace(None))
        torch.cuda.synchronize()
        t = tr.cpu().numpy().astype(np.float64)
        c = t[:148 * 8].reshape(148, 8)
        u = t[148 * 8:].reshape(148, 8, 8)
        t0 = c[c[:, 0] > 0, 0].min()
        print(f"== {label} split {sk}: span {(c[:, 7].max() - t0) / 1e3:.2f} us")
        for cta in (0, 1, 2, 3, 40, 41, 100, 101):
            row = []
            for it in range(8):
                if u[cta, it, 1] == 0:
                    continue
                row.append("u%d[" % it + " ".join(f"{ev[k][:4]}={(u[cta, it, k] - t0) / 1e3:.1f}"
                                                   for k in range(7) if u[cta, it, k] > 0) + "]")
            print(f"  cta {cta:3d}: " + "  ".join(row))
    lib.dart_gemm_force_splitk(1)
