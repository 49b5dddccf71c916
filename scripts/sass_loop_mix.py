"""Instruction mix of the hottest (largest backward-branch) loop of one kernel in a .so.
    python scripts/sass_loop_mix.py paper_2603_11441_b200/libdart_b200.so flash_attn_kernelILi16"""
import collections
import re
import subprocess
import sys

so, pat = sys.argv[1], sys.argv[2]
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
body = next(f for f in funcs if f.split("\n", 1)[0].find(pat) >= 0)
ins = []
for l in body.split("\n"):
    m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), l))
loops = []
for off, op, l in ins:
    if op == "BRA":
        t = re.search(r"0x([0-9a-f]+)", l.split("BRA", 1)[1])
        if t and int(t.group(1), 16) < off:
            loops.append((int(t.group(1), 16), off))
print(body.split("\n", 1)[0][:100], "| total instructions", len(ins))
for lo, hi in sorted(loops, key=lambda x: x[0] - x[1])[:2]:
    c = collections.Counter(op for off, op, _ in ins if lo <= off <= hi)
    print(f"loop {lo:#x}-{hi:#x}: {sum(c.values())} instructions")
    print("  " + ", ".join(f"{k} {v}" for k, v in c.most_common(30)))
