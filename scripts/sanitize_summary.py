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
    o.write("\nReading. memcheck and synccheck: 0 errors for every driver. racecheck: the only reports are in the\n"
            "CTA-pair GEMM instantiations (`gemm_heads_kernel<2, ...>`), one per launch, all of the form \"write at an\n"
            "unknown PC / read at the `tcgen05.alloc.cta_group::2` line\": the collective TMEM allocation of a CTA pair\n"
            "writes the allocated address into the `tmem_slot` word of BOTH CTAs' shared memory (a cross-CTA write\n"
            "the tool cannot attribute), and every thread reads that word only after the cluster barrier and a\n"
            "`__syncthreads()` (rk_gemm.cu, kernel prologue). The single-CTA instantiations (`RK_GEMM_CLUSTER=1`)\n"
            "and every other kernel (votes, averages, moments, serving, arrivals, fused path, actor-critic) report\n"
            "no hazard.\n")
print(open("profiles/r02_sanitizer.md").read())
