"""Opcode mix (executed warp instructions) and stall samples of an `ncu --page source --csv
--print-source sass` export, for instructions executed at least FRAC of the hottest one."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.3
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
isrc, iss, iex = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
num = lambda x: int(x) if x.strip().isdigit() else 0
tot = sum(num(r[iss]) for r in data)
mx = max(num(r[iex]) for r in data)
c, cs = Counter(), Counter()
allex = sum(num(r[iex]) for r in data)
for r in data:
    ex = num(r[iex])
    toks = r[isrc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    op = op.split(".")[0]
    if ex >= mx * frac:
        c[op] += ex
        cs[op] += num(r[iss])
hot = sum(c.values())
print(f"stall samples {tot}, executed warp-instr {allex}, hot set {hot} ({hot/allex:.0%})")
for k, v in c.most_common(40):
    print(f"{k:10s} {v:12d} {v/hot:6.1%}  stall samples {cs[k]:7d} ({cs[k]/max(tot,1):.1%})")
