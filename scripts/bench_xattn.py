"""Text cross-attention shape (hd 16, 32 text keys, class-shared image rows) through
dart_attention: N classes x 5184 query rows x 16 heads."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()
N, L, H, hd, Lt = int(sys.argv[1]) if len(sys.argv) > 1 else 80, 5184, 16, 16, 32
D = H * hd
q = torch.randn(N * L, D, device="cuda").half()
kv = torch.randn(N * Lt, 12 * D, device="cuda").half()  # 6 layers x (k | v), layer 0 used
o = torch.empty(N * L, D, device="cuda").half()
call = lambda: _native.check(lib.dart_attention(q.data_ptr(), kv.data_ptr(), kv[:, D:].data_ptr(), o.data_ptr(), N, H,
                                                L, Lt, hd, D, 12 * D, D, L * D, Lt * 12 * D, L * D, 0, 0,
                                                st.cuda_stream))
call()
torch.cuda.synchronize()
x = q.float().view(N, L, H, hd).transpose(1, 2)
k = kv[:, :D].float().view(N, Lt, H, hd).transpose(1, 2)
v = kv[:, D:2 * D].float().view(N, Lt, H, hd).transpose(1, 2)
ref = torch.softmax(x @ k.transpose(-1, -2) / hd ** 0.5, -1) @ v
err = (o.float().view(N, L, H, hd).transpose(1, 2) - ref).abs().max().item()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    call()
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 10 * 1000
print(f"text xattn N={N}: {t:.1f} us, max err {err:.2e}, {N * L * D * 2 * 2 / t / 1e3:.0f} GB/s (q read + o write)")
