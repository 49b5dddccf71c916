"""tcgen05 attention variants (DART_FA_VARIANT) at the DART shapes: correctness vs fp32 torch on
small items, then CUDA-event timing.  python scripts/bench_attn.py  (one variant per process)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2603_11441_b200 import _native

lib = _native.load()
st = torch.cuda.current_stream()


def run(qkv, o, items, H, L, hd):
    _native.check(lib.dart_attention_qkv(qkv.data_ptr(), o.data_ptr(), items, H, L, hd, None, st.cuda_stream))


def bench(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


var = os.environ.get("DART_FA_VARIANT", "0")
H = 16
for items, L, hd in [(2, 576, 80), (1, 5184, 80), (2, 5184, 16), (3, 576, 16)]:
    E = H * hd
    g = torch.Generator(device="cuda").manual_seed(L + items)
    qkv = (torch.randn(items, L, 3, H, hd, device="cuda", generator=g) * 2).half()
    o = torch.empty(items, L, E, device="cuda", dtype=torch.float16)
    run(qkv, o, items, H, L, hd)
    torch.cuda.synchronize()
    x = qkv.permute(2, 0, 3, 1, 4).float()
    ref = torch.softmax(x[0] @ x[1].transpose(-1, -2) / hd ** 0.5, -1) @ x[2]
    ref = ref.permute(0, 2, 1, 3).reshape(items, L, E)
    err = float((o.float() - ref).abs().max())
    print(f"var {var} check items={items} L={L} hd={hd}: max err {err:.2e} {'OK' if err < 1e-2 else 'FAIL'}")
for items, L, hd, name in [(1, 5184, 80, "bb global"), (9, 576, 80, "bb windowed"), (4, 5184, 16, "enc self N=4"),
                           (80, 5184, 16, "enc self N=80")]:
    E = H * hd
    qkv = torch.randn(items * L, 3 * E, device="cuda").half()
    o = torch.empty(items * L, E, device="cuda", dtype=torch.float16)
    t = bench(lambda: run(qkv, o, items, H, L, hd), 3 if items == 80 else 20)
    fl = 4 * items * H * L * L * hd
    print(f"var {var} {name:14s}: {t*1e3:9.1f} us {fl/t/1e9:7.1f} TF/s {items*H*L*L/t/1e6:8.1f} Gexp/s")
