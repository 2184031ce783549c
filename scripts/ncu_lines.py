"""Summarise an ncu report per CUDA source line: stall samples and executed instructions.

    python scripts/ncu_lines.py REPORT [TOP] [KERNEL_REGEX]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["-k", f"regex:{sys.argv[3]}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
his = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r]
agg, inst, src = collections.Counter(), collections.Counter(), {}
for n, hi in enumerate(his):
    h = rows[hi]
    ci, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    fname = ""
    for back in range(hi - 1, max(hi - 4, -1), -1):
        if rows[back] and rows[back][0] == "File Name":
            fname = rows[back][1].split("/")[-1]
            break
    end = his[n + 1] if n + 1 < len(his) else len(rows)
    for r in rows[hi + 1:end]:
        if len(r) < len(h) or not r[0] or not r[0].isdigit():
            continue
        try:
            key = f"{fname}:{r[0]}"
            agg[key] += int(r[ci]); inst[key] += int(r[ii] or 0); src[key] = r[1][:100]
        except ValueError:
            pass
tot = sum(agg.values()) or 1
print("total stall samples", tot, " instructions", sum(inst.values()))
for k, v in agg.most_common(top):
    print(f"{v:7d} {100 * v / tot:5.1f}% inst={inst[k]:>11d} {k}: {src[k]}")
