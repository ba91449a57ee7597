"""Summarise `nvcc -Xptxas -v` output: kernel (demangled, shortened), registers, spills, smem.

Usage: nvcc ... -Xptxas -v -c x.cu 2>&1 | python tools/ptxas_regs.py [regex]
"""
import re
import subprocess
import sys

pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
cur = None
rows = []
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line) or re.search(r"Function properties for (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        spill = int(m.group(1))
        rows.append([cur, None, spill, None])
    m = re.search(r"Used (\d+) registers.*?(\d+) bytes smem", line) or re.search(r"Used (\d+) registers", line)
    if m and cur and rows and rows[-1][0] == cur:
        rows[-1][1] = int(m.group(1))
        s = re.search(r"(\d+) bytes smem", line)
        rows[-1][3] = int(s.group(1)) if s else 0
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True, text=True).stdout.split("\n")
for r, n in zip(rows, names):
    n = re.sub(r"pmap::", "", n)
    n = re.sub(r"\(.*$", "", n)
    if pat and not pat.search(n):
        continue
    print(f"{r[1]!s:>4} regs {r[2]:>5} B spill {r[3]!s:>6} B smem  {n[:150]}")
