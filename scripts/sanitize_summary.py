"""Collect gpurun_out/san_<tool>_<shape>.log into profiles/r02_sanitizer.md."""
import glob
import os
import re

rows = []
for f in sorted(glob.glob("gpurun_out/san_*_*.log")):
    tool, shape = re.match(r".*san_(\w+?)_(\w+)\.log", f).groups()
    txt = open(f).read()
    summ = [ln for ln in txt.splitlines() if "SUMMARY" in ln]
    kern = sorted(set(re.findall(r"at void rk::<unnamed>::(\w+)", txt)))
    rows.append((tool, shape, summ[-1].replace("=========", "").strip() if summ else "no summary", ", ".join(kern)))
with open("profiles/r02_sanitizer.md", "w") as o:
    o.write("# compute-sanitizer, round 2\n\n`scripts/sanitize.sh` runs `compute-sanitizer --tool {memcheck,racecheck,synccheck}` over\n"
            "`scripts/sanitize_run.py {c1,c2,k12,fused,serve,rl}` (heads GEMM both tie modes, votes, averages, moments, predict;\n"
            "K = 12 averaging paths incl. caller logits and queue mode; the fused path with fallback; arrivals, greedy,\n"
            "async and stream serving; the actor-critic rollout / gradient / update).\n\n"
            "| tool | driver | summary | kernels named in reports |\n|---|---|---|---|\n")
    for r in rows:
        o.write(f"| {r[0]} | {r[1]} | {r[2]} | {r[3]} |\n")
print(open("profiles/r02_sanitizer.md").read())
