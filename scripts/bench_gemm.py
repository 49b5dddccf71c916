"""tcgen05 GEMM at the DART shapes (every epilogue) vs cuBLAS fp16 (torch.matmul), CUDA-event timed.
    python scripts/bench_gemm.py"""
import ctypes
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()
plan = os.environ.get("DART_GEMM_PLAN")
if plan:
    lib.dart_gemm_force_plan(*[int(x) for x in plan.split(",")])
if os.environ.get("DART_GEMM_SPLITK"):
    lib.dart_gemm_force_splitk(int(os.environ["DART_GEMM_SPLITK"]))


def bench(fn, reps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


T = 5184
inv = 100.0 ** (-torch.arange(20, dtype=torch.float64) / 20)
rr = torch.arange(72, dtype=torch.float64).repeat_interleave(72)
cc = torch.arange(72, dtype=torch.float64).repeat(72)
ang = torch.cat([rr[:, None] * inv, cc[:, None] * inv], 1)
cos, sin = torch.cos(ang).float().cuda().contiguous(), torch.sin(ang).float().cuda().contiguous()
print("GEMM  M x N x K  epi: ours us / TF/s | cuBLAS fp16 us / TF/s   plan", os.environ.get("DART_GEMM_PLAN", "auto"))
shapes = [(5184, 3840, 1280, 4, "qkv+rope"), (5184, 3840, 1280, 0, "qkv plain"), (5184, 1280, 1280, 3, "attn.out+res"),
          (5184, 5120, 1280, 1, "fc1+relu"), (5184, 1280, 5120, 3, "fc2+res"), (20736, 256, 256, 0, "enc q N=4"),
          (20736, 1024, 256, 1, "enc fc1 N=4"), (20736, 256, 1024, 3, "enc fc2 N=4"),
          (414720, 256, 256, 0, "enc q N=80"), (414720, 512, 256, 0, "enc kv N=80"), (414720, 1024, 256, 1, "enc fc1 N=80"),
          (414720, 256, 1024, 3, "enc fc2 N=80"), (414720, 256, 256, 3, "enc out N=80"), (414720, 3072, 256, 0, "dec kv N=80")]
sel = sys.argv[1:]
for (M, N, K, epi, name) in shapes:
    if sel and not any(s in name for s in sel):
        continue
    A = torch.randn(M, K, device="cuda").half()
    W = (torch.randn(N, K, device="cuda") / math.sqrt(K)).half()
    bias = torch.zeros(N, device="cuda")
    out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi in (2, 3) else torch.float16)
    rc, rs = (cos.data_ptr(), sin.data_ptr()) if epi == 4 else (None, None)
    f = lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None, M, N, K,
                                            epi, rc, rs, T, 80, 2560 if epi == 4 else 0, st.cuda_stream))
    t = bench(f)
    tc = bench(lambda: torch.matmul(A, W.T))
    fl = 2 * M * N * K
    bn, cg = ctypes.c_int32(), ctypes.c_int32()
    lib.dart_gemm_plan(M, N, epi, ctypes.byref(bn), ctypes.byref(cg))
    print(f"{name:14s} {M}x{N}x{K} e{epi}: {t*1e3:8.1f} us {fl/t/1e9:7.1f} | {tc*1e3:8.1f} us {fl/tc/1e9:7.1f}"
          f"   bn {bn.value} cg {cg.value}")
