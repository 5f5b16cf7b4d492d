"""Top SASS lines by warp-stall samples from an ncu report (host tool).

usage: python tools/ncu_hot.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
key = "Warp Stall Sampling (All Samples)"
body = [r for r in rows[2:] if len(r) == len(h)]
tot = sum(float(r[idx[key]] or 0) for r in body) or 1.0
print(f"{len(body)} SASS lines, {tot:.0f} samples")
for i, r in enumerate(body):
    r.append(i)
for r in sorted(body, key=lambda r: -float(r[idx[key]] or 0))[:top]:
    print(f"{float(r[idx[key]]) / tot * 100:5.1f}%  #{r[-1]:5d}  {r[idx['Source']].strip()[:100]}")
