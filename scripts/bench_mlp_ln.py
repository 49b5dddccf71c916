"""Fused enc-dec MLP with the next sub-block's LayerNorm (dart_mlp_fused_ln) at the N=4 and N=80 row
counts; prints us per launch and a checksum of the outputs (A/B across builds via DART_LIB_PATH)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream().cuda_stream
for M in (20736, 414720):
    g = torch.Generator(device="cuda").manual_seed(M)
    h = torch.randn(M, 256, device="cuda", generator=g).half()
    w1 = (torch.randn(1024, 256, device="cuda", generator=g) / 16).half()
    w2 = (torch.randn(256, 1024, device="cuda", generator=g) / 32).half()
    b1, b2 = torch.randn(1024, device="cuda", generator=g), torch.randn(256, device="cuda", generator=g)
    lg, lb = torch.rand(256, device="cuda", generator=g) + 0.5, torch.randn(256, device="cuda", generator=g)
    x0 = torch.randn(M, 256, device="cuda", generator=g)
    x = x0.clone()
    ho = torch.empty(M, 256, device="cuda").half()
    f = lambda: _native.check(lib.dart_mlp_fused_ln(h.data_ptr(), w1.data_ptr(), b1.data_ptr(), w2.data_ptr(),
                                                    b2.data_ptr(), x.data_ptr(), ho.data_ptr(), lg.data_ptr(),
                                                    lb.data_ptr(), M, st))
    f()
    torch.cuda.synchronize()
    ck = (float(x.double().sum()), float(ho.double().sum()))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"M={M}: {e0.elapsed_time(e1) / reps * 1000:8.1f} us  checksum x {ck[0]:.6f} h {ck[1]:.6f}")
