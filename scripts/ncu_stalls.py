"""Warp-stall breakdown of one kernel's SASS region from `ncu --page source --csv --print-source sass`.
    python scripts/ncu_stalls.py source.csv <kernel substring> [first_mnemonic_regex]
Prints per-kernel stall totals, then the hottest instructions with their dominant stalls."""
import csv
import re
import sys

path, pat = sys.argv[1], sys.argv[2]
kernels, cur = [], None
with open(path) as f:
    for row in csv.reader(f):
        if row and row[0] == "Kernel Name":
            cur = {"name": row[1], "rows": []}
            kernels.append(cur)
        elif row and row[0] == "Address":
            cur["hdr"] = row
        elif cur is not None and row:
            cur["rows"].append(row)
for k in kernels:
    if pat not in k["name"]:
        continue
    h = k["hdr"]
    ix = {n: i for i, n in enumerate(h)}
    stall_cols = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
    tot = {n: 0 for n in stall_cols}
    samples = 0
    rows = []
    for r in k["rows"]:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        samples += s
        st = {n: int(r[ix[n]] or 0) for n in stall_cols}
        for n in stall_cols:
            tot[n] += st[n]
        rows.append((s, r[ix["Address"]], r[ix["Source"]].strip(), st))
    print(k["name"][:110], "samples", samples)
    print("  " + ", ".join(f"{n[6:]} {v / max(1, samples):.1%}" for n, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
    for s, a, src, st in sorted(rows, key=lambda x: -x[0])[:25]:
        top = sorted(st.items(), key=lambda x: -x[1])[:3]
        print(f"  {s:6d} {a[-5:]} {src[:60]:60s} " + " ".join(f"{n[6:]}={v}" for n, v in top if v))
