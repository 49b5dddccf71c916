"""One warm + one profiled dart_gemm launch: python scripts/prof_gemm.py M N K epi [bn cg]"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
M, N, K, epi = (int(x) for x in sys.argv[1:5])
if len(sys.argv) > 6:
    lib.dart_gemm_force_plan(int(sys.argv[5]), int(sys.argv[6]))
A = torch.randn(M, K, device="cuda").half()
W = (torch.randn(N, K, device="cuda") / math.sqrt(K)).half()
bias = torch.zeros(N, device="cuda")
out = torch.zeros(M, N, device="cuda", dtype=torch.float32 if epi in (2, 3) else torch.float16)
st = torch.cuda.current_stream().cuda_stream
f = lambda: _native.check(lib.dart_gemm(A.data_ptr(), W.data_ptr(), bias.data_ptr(), out.data_ptr(), None, M, N, K, epi,
                                        None, None, 0, 0, 0, st))
f()
torch.cuda.synchronize()
torch.cuda.profiler.start()
f()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
