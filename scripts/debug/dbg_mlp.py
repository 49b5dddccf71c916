import sys, torch
sys.path.insert(0, '.')
from paper_2603_11441_b200 import _native
lib = _native.load(); st = torch.cuda.current_stream().cuda_stream
M = 512
g = torch.Generator(device="cuda").manual_seed(1)
h = torch.randn(M, 256, device="cuda", generator=g).half()
w1 = (torch.randn(1024, 256, device="cuda", generator=g) / 16).half()
w2 = (torch.randn(256, 1024, device="cuda", generator=g) / 32).half()
b1 = torch.zeros(1024, device="cuda"); b2 = torch.zeros(256, device="cuda")
x = torch.zeros(M, 256, device="cuda")
hid = torch.relu(h.float() @ w1.float().T + b1).half().float()
ref = x + hid @ w2.float().T + b2
out = x.clone()
_native.check(lib.dart_mlp_fused(h.data_ptr(), w1.data_ptr(), b1.data_ptr(), w2.data_ptr(), b2.data_ptr(), out.data_ptr(), M, st))
torch.cuda.synchronize()
d = (out - ref).abs()
print("max err", d.max().item(), "ref max", ref.abs().max().item())
print("err by row block (32 rows):", [round(d[i:i+32].max().item(), 3) for i in range(0, M, 32)])
print("err by col block (32 cols):", [round(d[:, i:i+32].max().item(), 3) for i in range(0, 256, 32)])
# test: only one hidden slice active
for e in range(8):
    w2m = torch.zeros_like(w2); w2m[:, e*128:(e+1)*128] = w2[:, e*128:(e+1)*128]
    out = x.clone()
    _native.check(lib.dart_mlp_fused(h.data_ptr(), w1.data_ptr(), b1.data_ptr(), w2m.data_ptr(), b2.data_ptr(), out.data_ptr(), M, st))
    torch.cuda.synchronize()
    r = hid @ w2m.float().T
    print("slice", e, "err", (out - r).abs().max().item(), "ref", r.abs().max().item(), "ratio", (out[:4,:4]/r[:4,:4]).flatten()[:4].tolist())
