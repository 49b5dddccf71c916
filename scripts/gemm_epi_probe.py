"""Epilogue cost of the N=1280 residual GEMM: the same M x N output with K = 64 (one k-block, so the
main loop is negligible) for each epilogue, and the full K, with the residual L2-warm (back-to-back) and
cold (a 256 MB buffer written between launches).  python scripts/gemm_epi_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()
flush = torch.empty(64 * 1024 * 1024, device="cuda")


def bench(fn, reps=30, cold=False):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if cold:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


M, N = 5184, 1280
for K in (64, 1280, 5120):
    A = torch.randn(M, K, device="cuda").half()
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).half()
    bias = torch.zeros(N, device="cuda")
    o32 = torch.zeros(M, N, device="cuda")
    o16 = torch.zeros(M, N, device="cuda", dtype=torch.float16)
    for bn, cg in ((256, 2), (256, 1)):
        lib.dart_gemm_force_plan(bn, cg)
        for epi, out in ((0, o16), (2, o32), (3, o32)):
            f = lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None,
                                                    M, N, K, epi, None, None, 0, 0, 0, st.cuda_stream))
            print(f"K={K:5d} bn {bn} cg {cg} epi {epi}: warm {bench(f):6.1f} us  cold {bench(f, cold=True):6.1f} us")
    lib.dart_gemm_force_plan(0, 0)
