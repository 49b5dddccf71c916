"""N=1280 backbone GEMMs (attn.out K=1280, mlp.fc2 K=5120): epilogue and tile-plan variants,
CUDA-event timed, against cuBLAS.  python scripts/gemm_n1280.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()


def bench(fn, reps=50):
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


M, N = 5184, 1280
for K in (1280, 5120):
    A = torch.randn(M, K, device="cuda").half()
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).half()
    bias = torch.zeros(N, device="cuda")
    o32 = torch.zeros(M, N, device="cuda")
    o16 = torch.zeros(M, N, device="cuda", dtype=torch.float16)
    fl = 2 * M * N * K
    tc = bench(lambda: torch.matmul(A, W.t()))
    print(f"K={K}: cuBLAS {tc:6.1f} us {fl / tc / 1e6:6.0f} TF/s")
    for bn, cg in ((0, 0), (256, 2), (128, 2), (256, 1), (128, 1), (64, 2)):
        lib.dart_gemm_force_plan(bn, cg)
        for epi, out in ((0, o16), (2, o32), (3, o32)):
            t = bench(lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(),
                                                           None, M, N, K, epi, None, None, 0, 0, 0, st.cuda_stream)))
            print(f"  plan bn {bn:3d} cg {cg}  epi {epi}: {t:6.1f} us {fl / t / 1e6:6.0f} TF/s")
    lib.dart_gemm_force_plan(0, 0)
    for sk in (2,):
        lib.dart_gemm_force_splitk(sk)
        t = bench(lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), o32.data_ptr(),
                                                       None, M, N, K, 3, None, None, 0, 0, 0, st.cuda_stream)))
        print(f"  split-K {sk} epi 3: {t:6.1f} us {fl / t / 1e6:6.0f} TF/s")
        lib.dart_gemm_force_splitk(1)
