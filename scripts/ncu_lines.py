"""Summarise an ncu report per CUDA source line: stall samples and executed instructions."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if "Warp Stall Sampling (All Samples)" in r]
h = rows[hi[0]]
ci, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
agg, inst, src = collections.Counter(), collections.Counter(), {}
end = hi[1] if len(hi) > 1 else len(rows)
for r in rows[hi[0] + 1:end]:
    if len(r) < len(h) or not r[0]:
        continue
    try:
        agg[r[0]] += int(r[ci]); inst[r[0]] += int(r[ii] or 0); src[r[0]] = r[1][:110]
    except ValueError:
        pass
tot = sum(agg.values()) or 1
print("total stall samples", tot, " instructions", sum(inst.values()))
for k, v in agg.most_common(top):
    print(f"{v:7d} {100 * v / tot:5.1f}% inst={inst[k]:>11d} L{k}: {src[k]}")
