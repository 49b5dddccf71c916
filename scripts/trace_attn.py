"""CTA-0 timeline of the tcgen05 attention (hd 16 encoder self-attention shape, N=4 classes):
clock64 stamps per key tile -> per-tile latencies of the S -> softmax -> P -> P.V chain."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()
hd = int(sys.argv[1]) if len(sys.argv) > 1 else 16
items, L, H = (4, 5184, 16) if hd == 16 else (1, 5184, 16)
E = H * hd
qkv = torch.randn(items * L, 3 * E, device="cuda").half()
o = torch.empty(items * L, E, device="cuda", dtype=torch.float16)
tr = torch.zeros(11 * 256, dtype=torch.int64, device="cuda")
run = lambda: _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o.data_ptr(), items, H, L, hd, None, st.cuda_stream))
run()
lib.dart_attention_trace(tr.data_ptr())
run()
torch.cuda.synchronize()
lib.dart_attention_trace(None)
t = tr.cpu().numpy().reshape(11, 256).astype(np.int64)
s_ready, p_done, p_seen, issued, v_ok, pv_issued, k_ok = t[:7]
pw = t[7:11]  # P done per softmax warp 2..5
if pw.any():
    print("per-warp P-done minus warp 2 (warps 3, 4, 5), tiles 10..30:")
    for g in range(10, 30):
        print(g, [int(pw[w][g] - pw[0][g]) for w in (1, 2, 3)])
base = s_ready[0]
print("tile  S_ready  P_done(soft)  P_seen(mma)  issued   | soft_work  mma_react  issue  S_gap")
for g in range(1, 40):
    print(f"{g:4d} {s_ready[g]-base:8d} {p_done[g]-base:10d} {p_seen[g]-base:11d} {issued[g]-base:8d}   | "
          f"{p_done[g]-s_ready[g]:8d} {p_seen[g]-p_done[g]:9d} {issued[g]-p_seen[g]:6d} {s_ready[g]-s_ready[g-1]:6d}")
print("tile | p_seen->v_ok  v_ok->pv_issued  pv_issued->k_ok(next S)  k_ok->issued")
for g in range(10, 30):
    print(f"{g:4d} | {v_ok[g]-p_seen[g]:8d} {pv_issued[g]-v_ok[g]:10d} {k_ok[g]-pv_issued[g]:12d} {issued[g]-k_ok[g]:10d}")
d = np.diff(s_ready[10:200])
print("median tile period", np.median(d), "softmax work median", np.median((p_done - s_ready)[10:200]),
      "S wait (S_ready - prev P_done) median", np.median((s_ready[11:200] - p_done[10:199])))
