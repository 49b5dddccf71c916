"""Enc-dec MLP: fused kernel (dart_mlp_fused) vs fc1 + fc2 GEMMs (dart_gemm), N=4 and N=80 rows."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream().cuda_stream


def bench(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000


for M in (20736, 414720):
    h = torch.randn(M, 256, device="cuda").half()
    w1 = (torch.randn(1024, 256, device="cuda") / 16).half()
    w2 = (torch.randn(256, 1024, device="cuda") / 32).half()
    b1, b2 = torch.zeros(1024, device="cuda"), torch.zeros(256, device="cuda")
    x = torch.randn(M, 256, device="cuda")
    hid = torch.empty(M, 1024, device="cuda").half()
    fused = lambda: _native.check(lib.dart_mlp_fused(h.data_ptr(), w1.data_ptr(), b1.data_ptr(), w2.data_ptr(),
                                                     b2.data_ptr(), x.data_ptr(), M, st))

    def unfused():
        _native.check(lib.dart_gemm(h.data_ptr(), w1.data_ptr(), b1.data_ptr(), hid.data_ptr(), None, M, 1024, 256, 1,
                                    None, None, 0, 0, 0, st))
        _native.check(lib.dart_gemm(hid.data_ptr(), w2.data_ptr(), b2.data_ptr(), x.data_ptr(), None, M, 256, 1024, 3,
                                    None, None, 0, 0, 0, st))
    tf, tu = bench(fused), bench(unfused)
    fl = 4 * M * 256 * 1024
    print(f"MLP M={M}: fused {tf:8.1f} us ({fl / tf / 1e6:6.0f} TF/s) | fc1+fc2 GEMMs {tu:8.1f} us ({fl / tu / 1e6:6.0f} TF/s)")
