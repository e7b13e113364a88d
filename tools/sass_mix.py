"""Instruction mix per output from an ncu SASS source export: python tools/sass_mix.py file outputs"""
import collections
import csv
import signal
import sys

signal.signal(signal.SIGPIPE, signal.SIG_DFL)  # quiet when piped into head

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
i_src, i_ex = hdr.index("Source"), hdr.index("Instructions Executed")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
n_out = float(sys.argv[2]) / 32.0  # warp-level outputs
ops, stalls = collections.Counter(), collections.Counter()
for x in data:
    ex = int(x[i_ex] or 0)
    toks = x[i_src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    ops[op.split(".")[0]] += ex
    stalls[op.split(".")[0]] += int(x[i_s] or 0)
tot = sum(ops.values())
print(f"total warp-instructions {tot}, per output {tot / n_out:.2f}")
for op, n in ops.most_common(25):
    print(f"{op:12s} {n / n_out:6.2f} per output   stall share {stalls[op] / max(1, sum(stalls.values())):.1%}")
