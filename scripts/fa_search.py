"""Placement search for the FMA-pipe polynomial exponentials of the hd-16 softmax (variants 100+ of a
-DDART_FA_SEARCH build, see csrc/attention_search.inc): enc self-attention N=20, interleaved rounds,
median per variant; the top variants re-timed against production and checked against it.
    DART_LIB_PATH=build/lib_search.so python scripts/fa_search.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()
masks = {int(k): v for k, v in json.load(open(os.path.join(os.path.dirname(__file__), "fa_search_masks.json"))).items()}
items, L, hd = 20, 5184, 16
qkv = torch.randn(items * L, 3 * 16 * hd, device="cuda").half()
o = torch.empty(items * L, 16 * hd, device="cuda").half()


def run():
    _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o.data_ptr(), items, 16, L, hd, None, st.cuda_stream))


def timed(reps):
    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000.0


vs = [0] + sorted(masks)
res = {v: [] for v in vs}
for rnd in range(3):
    for v in vs:
        lib.dart_attention_variant(v)
        res[v].append(timed(3))
med = {v: float(np.median(t)) for v, t in res.items()}
rank = sorted(masks, key=lambda v: med[v])
print(f"production (first 3 of 8 pairs): {med[0]:.1f} us")
for v in rank[:12]:
    print(f"  v{v} mask {masks[v]:08b} ({bin(masks[v]).count('1')} of 8 pairs): {med[v]:.1f} us")
print("worst:", ", ".join(f"{masks[v]:08b} {med[v]:.0f}" for v in rank[-5:]))
# re-time the best 6 against production, interleaved, and check them
top = [0] + rank[:6]
res2 = {v: [] for v in top}
for rnd in range(7):
    for v in top:
        lib.dart_attention_variant(v)
        res2[v].append(timed(5))
lib.dart_attention_variant(0)
run()
torch.cuda.synchronize()
ref = o.float().clone()
for v in top:
    lib.dart_attention_variant(v)
    run()
    torch.cuda.synchronize()
    d = (o.float() - ref).abs().max().item()
    print(f"re-timed v{v} mask {masks.get(v, 7):08b}: {np.median(res2[v]):.1f} us, max |diff| vs production {d:.2e}")
lib.dart_attention_variant(0)
