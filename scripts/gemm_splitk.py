"""Split-K (two K halves per tile, partial-accumulator combine) vs one unit per tile on the
backbone GEMM shapes at one image (M = 5184), CUDA-event timed back to back, against cuBLAS.
    python scripts/gemm_splitk.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()


def bench(fn, reps=100):
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


M = 5184
for name, N, K, epi in (("attn.qkv", 3840, 1280, 0), ("attn.out", 1280, 1280, 3), ("mlp.fc1", 5120, 1280, 1),
                        ("mlp.fc2", 1280, 5120, 3)):
    A = torch.randn(M, K, device="cuda").half()
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).half()
    bias = torch.zeros(N, device="cuda")
    out = torch.zeros(M, N, device="cuda", dtype=torch.float16 if epi in (0, 1) else torch.float32)
    fl = 2 * M * N * K
    tc = bench(lambda: torch.matmul(A, W.t()))
    line = f"{name:9s} M={M} N={N} K={K} epi {epi}: cuBLAS {tc:6.1f} us ({fl / tc / 1e6:5.0f} TF/s)"
    for sk in (1, 2):
        lib.dart_gemm_force_splitk(sk)
        t = bench(lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(),
                                                       None, M, N, K, epi, None, None, 0, 0, 0, st.cuda_stream)))
        line += f" | split {sk}: {t:6.1f} us ({fl / t / 1e6:5.0f} TF/s)"
    lib.dart_gemm_force_splitk(1)
    print(line, flush=True)
