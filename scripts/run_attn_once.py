"""One tcgen05 attention launch at a DART shape (for ncu captures).
    python scripts/run_attn_once.py ITEMS L HD [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
items, L, hd = (int(x) for x in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
H = 16
qkv = torch.randn(items * L, 3 * H * hd, device="cuda").half()
o = torch.empty(items * L, H * hd, device="cuda", dtype=torch.float16)
st = torch.cuda.current_stream()
for _ in range(reps):
    _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o.data_ptr(), items, H, L, hd, None, st.cuda_stream))
torch.cuda.synchronize()
print("ok")
