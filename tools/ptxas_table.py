"""Summarise `nvcc -Xptxas -v` output: kernel (demangled) | registers | spills | smem."""
import re
import subprocess
import sys

text = sys.stdin.read()
rows = []
cur = None
for line in text.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur["spill"] = int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
names = [r["name"] for r in rows]
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
filt = sys.argv[1] if len(sys.argv) > 1 else ""
for r, d in zip(rows, dem):
    d = d.replace("pmap::", "")
    if filt and not re.search(filt, d):
        continue
    print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill', '?'):>5}  {d[:150]}")
