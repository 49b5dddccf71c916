"""In-process A/B of tcgen05 attention variants (interleaved rounds, median per variant), so
box-to-box clock / power-cap variation cancels.  python scripts/ab_attn.py 0 1 [2 ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()
variants = [int(v) for v in sys.argv[1:]] or [0, 1]
shapes = [(1, 5184, 80, "bb global"), (9, 576, 80, "bb windowed"), (20, 5184, 16, "enc self N=20")]
bufs = {}
for items, L, hd, name in shapes:
    E = 16 * hd
    bufs[name] = (torch.randn(items * L, 3 * E, device="cuda").half(), torch.empty(items * L, E, device="cuda").half())


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000.0


res = {(v, n): [] for v in variants for *_, n in shapes}
for rnd in range(5):
    for v in variants:
        lib.dart_attention_variant(v)
        for items, L, hd, name in shapes:
            qkv, o = bufs[name]
            res[(v, name)].append(timed(lambda: _native.check(lib.dart_attention_qkv(
                qkv.data_ptr(), o.data_ptr(), items, 16, L, hd, None, st.cuda_stream)), 10 if items < 10 else 4))
for *_, name in shapes:
    print(name, "  ".join(f"v{v}: {np.median(res[(v, name)]):8.1f} us" for v in variants))
# agreement with the first variant (same inputs)
ref = {}
for v in variants:
    lib.dart_attention_variant(v)
    for items, L, hd, name in shapes:
        qkv, o = bufs[name]
        _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o.data_ptr(), items, 16, L, hd, None, st.cuda_stream))
        torch.cuda.synchronize()
        if v == variants[0]:
            ref[name] = o.float().clone()
        else:
            print(f"v{v} {name}: max |diff| vs v{variants[0]} = {(o.float() - ref[name]).abs().max().item():.3e}")
lib.dart_attention_variant(0)
