"""Per-tile epilogue cost: K = 64 GEMMs (one k-block) with 1, 2, 3, 4 tiles per CTA pair
(M = 256 x 14 / 29 / 44 / 59 rows x N 1280 -> 70 / 145 / 220 / 295 tiles of 256 x 256 on 74 pairs),
back-to-back launches (launch gaps hidden), per epilogue.  python scripts/gemm_epi_probe2.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()


def bench(fn, reps=40):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


N, K = 1280, int(os.environ.get("K", "64"))
lib.dart_gemm_force_plan(256, 2)
for rb in (14, 29, 44, 59):
    M = 256 * rb
    A = torch.randn(M, K, device="cuda").half()
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).half()
    bias = torch.zeros(N, device="cuda")
    o32 = torch.zeros(M, N, device="cuda")
    o16 = torch.zeros(M, N, device="cuda", dtype=torch.float16)
    res = []
    for epi, out in ((0, o16), (2, o32), (3, o32)):
        f = lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None,
                                                M, N, K, epi, None, None, 0, 0, 0, st.cuda_stream))
        res.append(f"epi {epi}: {bench(f):6.2f} us")
    print(f"K={K} M={M:6d} tiles={rb * 5:4d}  " + "  ".join(res))
lib.dart_gemm_force_plan(0, 0)
