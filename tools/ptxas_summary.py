"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spills (reads stdin)."""
import re
import subprocess
import sys

cur = None
rows = []
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = (int(m.group(1)), int(m.group(2)), int(m.group(3)))
        rows.append([cur, spill])
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and rows and rows[-1][0] == cur and len(rows[-1]) == 2:
        rows[-1].append(int(m.group(1)))
names = subprocess.run(["c++filt"], input="\n".join(r[0] for r in rows), capture_output=True,
                       text=True).stdout.splitlines()
for n, r in zip(names, rows):
    n = n.replace("prngd::", "").replace("(CUtensorMap_st, GenArgs)", "")
    print(f"{r[2] if len(r) > 2 else '?':>4} regs  stack/spill {r[1]}  {n}")
