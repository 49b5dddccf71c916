"""Fixed per-launch cost of the persistent GEMM: back-to-back launches of tiny problems (one or a
few tiles, K = 64), PDL on and off; plus the LayerNorm and an empty torch kernel for scale.
    python scripts/gemm_fixed_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()


def bench(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


x = torch.zeros(16, device="cuda")
print(f"torch x.add_(1) (launch floor): {bench(lambda: x.add_(1)):6.2f} us")
for pdl in (1, 0):
    lib.dart_set_pdl(pdl)
    for M, N, K, epi in ((256, 256, 64, 0), (256 * 74, 256, 64, 0), (256, 256, 64, 3), (256 * 74, 256, 1280, 0),
                         (256 * 74, 256, 1280, 3)):
        A = torch.randn(M, K, device="cuda").half()
        W = torch.randn(N, K, device="cuda").half()
        bias = torch.zeros(N, device="cuda")
        out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi == 3 else torch.float16)
        f = lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None,
                                                M, N, K, epi, None, None, 0, 0, 0, st.cuda_stream))
        print(f"pdl {pdl} gemm M={M:6d} N={N} K={K:5d} epi {epi}: {bench(f):7.2f} us")
lib.dart_set_pdl(-1)
