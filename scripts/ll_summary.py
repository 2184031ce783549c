"""Per-kernel totals of an ncu launch list (gpu__time_duration.sum CSV): python scripts/ll_summary.py FILE [STEPS]

Prints each kernel's launch count and mean duration; with STEPS, the mean per step over the whole list."""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[start + 1:]:
    if len(r) != len(h):
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "").split("::")[-1]
    d = agg.setdefault(name, [])
    d.append(float(r[vi].replace(",", "")) / 1e6)
for k, v in agg.items():
    print(f"{k[:60]:60s} n={len(v):3d} mean={sum(v) / len(v):8.3f} ms  min={min(v):8.3f}  max={max(v):8.3f}")
