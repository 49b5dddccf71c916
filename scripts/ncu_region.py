"""Print SASS lines of one kernel around given addresses (suffix match) with sample counts.
    python scripts/ncu_region.py source.csv <kernel substring> <addr_suffix> [before] [after]"""
import csv
import sys

path, pat, addr = sys.argv[1], sys.argv[2], sys.argv[3].lower()
before = int(sys.argv[4]) if len(sys.argv) > 4 else 12
after = int(sys.argv[5]) if len(sys.argv) > 5 else 6
rows, hdr, cur = [], None, None
with open(path) as f:
    for row in csv.reader(f):
        if row and row[0] == "Kernel Name":
            cur = pat in row[1]
        elif row and row[0] == "Address":
            hdr = {n: i for i, n in enumerate(row)}
        elif cur and row:
            rows.append(row)
for i, r in enumerate(rows):
    if r[hdr["Address"]].lower().endswith(addr):
        for r2 in rows[max(0, i - before): i + after]:
            print(f"{r2[hdr['Address']][-5:]} {int(r2[hdr['Warp Stall Sampling (All Samples)']] or 0):6d}  {r2[hdr['Source']].strip()[:90]}")
        break
