"""SASS evidence for the hot K1 (k_spmv_tma<CgSpmvOp<false,false>, 7>):
instruction mix, the TMA bulk copies / L2 bulk prefetches / mbarrier ops,
where the DFMAs live (IEEE div/sqrt slow paths only), and the software-
pipelined gather loop (LDG gathers + DMUL/DADD, no DFMA).  Writes markdown
to stdout: python scripts/sass_excerpt.py > profiles/r02_sass_k1.md"""
import re
import subprocess
import sys
from collections import Counter

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2306_17801_b200/lib/librvk.so"
FN = "_ZN3rvk10k_spmv_tmaINS_8CgSpmvOpILb0ELb0EEELi7EEEvNS_8SpmvArgsET_NS_8TailArgsE"
sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
lines = sass.split("\n")
s = next(i for i, l in enumerate(lines) if "Function : " + FN in l)
e = next((i for i in range(s + 1, len(lines)) if "Function :" in lines[i]), len(lines))
body = [l for l in lines[s:e] if re.search(r"/\*[0-9a-f]{4}\*/", l)]
pat = re.compile(r"/\*([0-9a-f]{4})\*/\s+((?:@!?U?P\w+\s+)?)([A-Z0-9_]+)([^;]*);")
ins = []
for l in body:
    m = pat.search(l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip(), m.group(3), m.group(4).strip()))
mix = Counter(op for _, _, op, _ in ins)
print(f"# SASS of the hot K1 ({FN})\n")
print(f"`cuobjdump -sass {LIB}` (sm_100a), {len(ins)} instructions.\n")
print("| op | count |\n|---|---|")
for op in ["UBLKCP", "UBLKPF", "SYNCS", "LDG", "LDS", "STG", "DMUL", "DADD", "DFMA", "MUFU"]:
    print(f"| {op} | {mix.get(op, 0)} |")
print("\n## TMA bulk copies, L2 bulk prefetches, mbarrier ops\n```")
for a, p, op, rest in ins:
    if op in ("UBLKCP", "UBLKPF") or op == "SYNCS":
        print(f"/*{a:04x}*/ {p} {op} {rest}".replace("  ", " "))
print("```")
# DFMA locations: contiguous runs (the div/sqrt subroutines called from the tails)
runs, cur = [], None
for a, p, op, rest in ins:
    if op == "DFMA":
        if cur and a - cur[1] <= 0x100:
            cur[1] = a
            cur[2] += 1
        else:
            cur = [a, a, 1]
            runs.append(cur)
print("\n## DFMA locations (address ranges)\n")
for a, b, n in runs:
    print(f"- 0x{a:04x}-0x{b:04x}: {n} DFMA")
# the gather loop: the densest window of LDG + DMUL without DFMA
best = None
for i in range(len(ins)):
    j = i
    nl = nm = 0
    while j < len(ins) and ins[j][0] - ins[i][0] < 0x600:
        nl += ins[j][2] == "LDG"
        nm += ins[j][2] == "DMUL"
        j += 1
    if any(ins[k][2] == "DFMA" for k in range(i, j)):
        continue
    if best is None or nl + nm > best[0]:
        best = (nl + nm, i, j)
_, i, j = best
print("\n## The gather loop (densest LDG + DMUL window, no DFMA)\n```")
for a, p, op, rest in ins[i:j]:
    print(f"/*{a:04x}*/ {p} {op} {rest}".replace("  ", " "))
print("```")
