"""LayerNorm at the DART shapes (backbone 5184 x 1280, enc-dec N=80 414720 x 256), CUDA-event timed.
DART_LN_WARPS / DART_LN_RPW select the launch shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream().cuda_stream
for rows, dim in [(5184, 1280), (20736, 256), (414720, 256)]:
    x = torch.randn(rows, dim, device="cuda")
    g, b = torch.ones(dim, device="cuda"), torch.zeros(dim, device="cuda")
    y = torch.empty(rows, dim, device="cuda", dtype=torch.float16)
    f = lambda: _native.check(lib.dart_layernorm(x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(), rows, dim, 1, st))
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        f()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 * 1000
    print(f"LN {rows}x{dim} warps={os.environ.get('DART_LN_WARPS', 8)} rpw={os.environ.get('DART_LN_RPW', 1)}: "
          f"{t:7.1f} us  {rows * dim * 6 / t / 1e3:6.0f} GB/s")
