"""Kernel microbenchmarks on the B200: tcgen05 GEMM vs cuBLAS (torch.matmul) on the DART
shapes, and the flash attention at the DART shapes.  CUDA-event timed, warm."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
torch.backends.cuda.matmul.allow_tf32 = False
st = torch.cuda.current_stream()


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


print("GEMM  M x N x K  epi: ours us / TF/s | cuBLAS fp16 us / TF/s")
for (M, N, K, epi, name) in [(5184, 3840, 1280, 0, "qkv"), (5184, 1280, 1280, 3, "attn.out"), (5184, 5120, 1280, 1, "fc1"),
                             (5184, 1280, 5120, 3, "fc2"), (20736, 256, 256, 0, "encq N=4"), (20736, 1024, 256, 1, "enc fc1 N=4"),
                             (20736, 256, 1024, 3, "enc fc2 N=4"), (20736, 3072, 256, 0, "dec kv-all N=4"),
                             (414720, 256, 256, 0, "encq N=80"), (414720, 1024, 256, 1, "enc fc1 N=80")]:
    A = torch.randn(M, K, device="cuda").half()
    W = (torch.randn(N, K, device="cuda") / math.sqrt(K)).half()
    bias = torch.zeros(N, device="cuda")
    out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi in (2, 3) else torch.float16)
    f = lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None, M, N, K,
                                            epi, None, None, 0, 0, 0, st.cuda_stream))
    t = bench(f)
    tc = bench(lambda: torch.matmul(A, W.T))
    fl = 2 * M * N * K
    print(f"{name:16s} {M}x{N}x{K} e{epi}: {t*1e3:8.1f} us {fl/t/1e9:7.1f} | {tc*1e3:8.1f} us {fl/tc/1e9:7.1f}")

print("ATTN tcgen05 (packed QKV)  items L: us  TF/s  Gexp/s")
for (items, L, name) in [(1, 5184, "bb global"), (9, 576, "bb windowed")]:
    H, hd = 16, 80
    E = H * hd
    qkv = torch.randn(items * L, 3 * E, device="cuda").half()
    o = torch.empty(items * L, E, device="cuda", dtype=torch.float16)
    f = lambda: _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o.data_ptr(), items, H, L, hd, None, st.cuda_stream))
    t = bench(f, reps=20)
    fl = 4 * items * H * L * L * hd
    print(f"{name:16s} {items} {L}: {t*1e3:9.1f} us {fl/t/1e9:7.1f} TF/s {items*H*L*L/t/1e6:8.1f} Gexp/s")

print("ATTN  batch heads Lq Lk hd: us  TF/s  Gexp/s")
for (B, H, Lq, Lk, hd, name) in [(1, 16, 5184, 5184, 80, "bb global"), (9, 16, 576, 576, 80, "bb windowed"),
                                  (4, 16, 5184, 5184, 16, "enc self N=4"), (4, 16, 5184, 32, 16, "enc text N=4"),
                                  (4, 16, 201, 5184, 16, "dec cross N=4"), (80, 16, 5184, 5184, 16, "enc self N=80")]:
    q = torch.randn(B, Lq, H, hd, device="cuda").half()
    k = torch.randn(B, Lk, H, hd, device="cuda").half()
    v = torch.randn(B, Lk, H, hd, device="cuda").half()
    o = torch.empty_like(q)
    E = H * hd
    f = lambda: _native.check(lib.dart_attention(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), B, H, Lq, Lk, hd,
                                                 E, E, E, Lq * E, Lk * E, Lq * E, 0, 0, st.cuda_stream))
    t = bench(f, reps=10)
    fl = 4 * B * H * Lq * Lk * hd
    print(f"{name:16s} {B} {H} {Lq} {Lk} {hd}: {t*1e3:9.1f} us {fl/t/1e9:7.1f} TF/s {B*H*Lq*Lk/t/1e6:8.1f} Gexp/s")
