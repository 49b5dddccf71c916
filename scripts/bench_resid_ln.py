"""Enc-dec residual GEMM with the fused LayerNorm epilogue (dart_gemm_resid_ln, K = 256, N = 256) at the
N=4 and N=80 row counts; us per launch and an output checksum (A/B across builds via DART_LIB_PATH)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream().cuda_stream
for M in (20736, 414720):
    g = torch.Generator(device="cuda").manual_seed(M + 1)
    A = torch.randn(M, 256, device="cuda", generator=g).half()
    W = (torch.randn(256, 256, device="cuda", generator=g) / 16).half()
    b = torch.randn(256, device="cuda", generator=g)
    lg, lb = torch.rand(256, device="cuda", generator=g) + 0.5, torch.randn(256, device="cuda", generator=g)
    x = torch.randn(M, 256, device="cuda", generator=g)
    h = torch.empty(M, 256, device="cuda").half()
    f = lambda: _native.check(lib.dart_gemm_resid_ln(A.data_ptr(), W.data_ptr(), b.data_ptr(), x.data_ptr(), h.data_ptr(),
                                                     lg.data_ptr(), lb.data_ptr(), M, 256, st))
    f()
    torch.cuda.synchronize()
    ck = float(h.double().sum())
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"resid+LN M={M}: {e0.elapsed_time(e1) / 20 * 1000:8.1f} us  checksum h {ck:.6f}")
