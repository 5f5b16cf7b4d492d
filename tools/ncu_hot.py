"""Top SASS lines by warp-stall samples from an ncu report (host tool).

usage: python tools/ncu_hot.py report.ncu-rep [top] [kernel-regex]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
flt = ["-k", "regex:" + sys.argv[3]] if len(sys.argv) > 3 else []
out = subprocess.run(["ncu", "-i", rep, *flt, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
key = "Warp Stall Sampling (All Samples)"
def num(x):
    try:
        float(x or 0)
        return True
    except ValueError:
        return False


body = [r for r in rows[2:] if len(r) == len(h) and num(r[idx[key]])]
tot = sum(float(r[idx[key]] or 0) for r in body) or 1.0
print(f"{len(body)} SASS lines, {tot:.0f} samples")
for i, r in enumerate(body):
    r.append(i)
for r in sorted(body, key=lambda r: -float(r[idx[key]] or 0))[:top]:
    print(f"{float(r[idx[key]]) / tot * 100:5.1f}%  #{r[-1]:5d}  {r[idx['Source']].strip()[:100]}")
