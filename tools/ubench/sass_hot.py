"""Summarise an ncu source page (SASS): instruction mix weighted by executions and stall samples."""
import csv
import io
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot_exec = 0
mix = Counter()
stall = Counter()
samples = []
for r in rows:
    src = r["Source"].strip()
    n = int(r["Instructions Executed"] or 0)
    s = int(r["Warp Stall Sampling (All Samples)"] or 0)
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    tot_exec += n
    mix[op] += n
    stall[op] += s
    samples.append((s, n, r["Address"][-5:], src[:80]))
tot_s = sum(stall.values())
print(f"total warp-instructions executed: {tot_exec:,}  stall samples: {tot_s:,}")
print("op mix (executed share, stall-sample share):")
for op, n in mix.most_common(25):
    print(f"  {op:10s} {n / tot_exec:6.1%}  {stall[op] / max(tot_s, 1):6.1%}")
print(f"top {top} instructions by stall samples:")
for s, n, a, src in sorted(samples, reverse=True)[:top]:
    print(f"  {s:6d} {n:10d} {a} {src}")
