"""Summarise the round's ncu artefacts (gpurun_out/<R>_*) into profiles/<R>_*.md / .json (committed)."""
import collections
import csv
import json
import re
import subprocess
import sys

R = sys.argv[1] if len(sys.argv) > 1 else "r01"
OUT = "profiles"


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    return name.split("::")[-1]


# ---- launch list of the bench command ------------------------------------------------------
rows = [r for r in csv.reader(open(f"gpurun_out/{R}_launches.csv")) if len(r) == 15 and r[0] != "ID"]
per = collections.OrderedDict()
for r in rows:
    k = short(r[4])
    d = per.setdefault(k, [0, 0.0])
    d[0] += 1
    d[1] += float(r[14]) / 1e6
ours = {"gemm_heads_kernel", "vote_classify_kernel", "vote_average_kernel", "vote_batch", "vote_cta", "vote_wsample",
        "vote_pair", "overdue_kernel", "merge_kernel", "q_kernel", "q_nested_kernel", "fold_kernel",
        "arrival_psum_kernel", "vote_sparse", "gather_rows", "queue_scan"}
tot_ours = sum(v[1] for k, v in per.items() if any(k.startswith(o) for o in ours))
lines = [f"# {R} launch list: `ncu --metrics gpu__time_duration.sum --clock-control none` of",
         "`python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1`",
         "", "Cold-cache, serialised per-launch times (compare SHARES, not absolutes). Raw CSV: "
         f"`{R}_launches.csv`.", "", "| kernel | launches | total ms | ms/launch | share of our kernels |",
         "|---|---|---|---|---|"]
for k, (n, ms) in per.items():
    ours_k = any(k.startswith(o) for o in ours)
    share = f"{100 * ms / tot_ours:.1f} %" if ours_k else "(harness)"
    lines.append(f"| {k} | {n} | {ms:.3f} | {ms / n:.3f} | {share} |")
open(f"{OUT}/{R}_launches.md", "w").write("\n".join(lines) + "\n")
subprocess.run(["cp", f"gpurun_out/{R}_launches.csv", f"{OUT}/{R}_launches.csv"])


# ---- --set full captures ----------------------------------------------------------------------
def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(out.splitlines()))
    hdr, units = rr[0], rr[1]
    res = []
    for r in rr[2:]:
        res.append({h: (f"{v} {u}".strip() if u else v) for h, v, u in zip(hdr, r, units)})
    return res


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "launch__grid_size", "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]
summary = {}
for tag in ("gemm", "vote", "k12", "gemm12", "fused"):
    try:
        recs = raw(f"gpurun_out/{R}_{tag}.ncu-rep")
    except Exception as e:  # noqa: BLE001
        print("skip", tag, e)
        continue
    for rec in recs:
        name = short(rec.get("Kernel Name", "?"))
        d = {}
        for w in WANT:
            for k, v in rec.items():
                if k.startswith(w):
                    d[k] = v
        key = f"{tag}:{name}"
        if key in summary:  # (the fused capture holds two GEMM instantiations / repeated kernels)
            key += f"#{sum(1 for k in summary if k.startswith(key))}"
        summary[key] = d
json.dump(summary, open(f"{OUT}/{R}_ncu_full.json", "w"), indent=1)
print(open(f"{OUT}/{R}_launches.md").read())
for k, d in summary.items():
    print(k)
    for kk, vv in d.items():
        print("   ", kk, vv)

# ---- DRAM traffic per launch for bench.py's roofline.traffic (scaled linearly in N to c4) ----------
CAPN = {"gemm": 65536, "vote": 200000, "k12": 250000, "gemm12": 131072, "fused": 131072}  # N of the captures
per_sample = {}
fused_ps = {"gemm": 0.0, "vote": 0.0, "fallback": 0.0}  # NEXT-3 path: fused GEMM, classify + sparse, fallback
for key, d in summary.items():
    tag, name = key.split(":", 1)
    if tag == "fused":
        b = 0.0
        for mk in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            val, unit = d.get(mk, "0 byte").split()[:2]
            b += float(val) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[unit] / CAPN["fused"]
        part = ("gemm" if name.startswith("gemm_heads_kernel<2, 0, 1>")
                else "vote" if name.startswith(("vote_classify", "vote_sparse")) else "fallback")
        fused_ps[part] += b
        continue
    if tag in ("k12", "gemm12"):
        continue  # c5 shape: reported in the summary, not part of the c4 traffic figure
    rd = float(d.get("dram__bytes_read.sum", "0 byte").split()[0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[
        d.get("dram__bytes_read.sum", "0 byte").split()[1]]
    wr = float(d.get("dram__bytes_write.sum", "0 byte").split()[0]) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[
        d.get("dram__bytes_write.sum", "0 byte").split()[1]]
    per_sample[name] = (rd + wr) / CAPN[tag]
k12_ps = 0.0  # c5 shape (K = 12, C = 100): the vote stage's kernels, scaled to c5's N = 4M
for key, d in summary.items():
    tag, name = key.split(":", 1)
    if tag != "k12":
        continue  # (the c5 GEMM capture gemm12 is summarised, its traffic not used by bench.py)
    for mk in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        val, unit = d.get(mk, "0 byte").split()[:2]
        k12_ps += float(val) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1}[unit] / CAPN["k12"]
gemm_ps = sum(v for k, v in per_sample.items() if k.startswith("gemm_heads"))
vote_ps = sum(v for k, v in per_sample.items() if k.startswith("vote_"))
tj = {"_note": f"DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch from the `ncu --set full` "
               f"captures of {R} (profiles/{R}_ncu_full.json; GEMM at N={CAPN['gemm']}, vote kernels at N={CAPN['vote']}, "
               f"K=8, C=1000, D=2048), scaled linearly in N to the c4 workload (N=1,000,000); c5: the K=12 vote kernels of the k12 capture "
               f"(N={CAPN['k12']}) scaled to N=4,000,000. vote_subsets = "
               f"classify + average kernels. Algorithmic: GEMM 36,096 B/sample (X 4,096 + fp32 logits 32,000), "
               f"vote 32,004 B/sample.",
      "c4": {"gemm_heads_tcgen05": round(gemm_ps * 1e6), "vote_subsets": round(vote_ps * 1e6)},
      "c5": {"vote_subsets": round(k12_ps * 4e6)},
      "c4_fused": {"gemm_heads_tcgen05": round(fused_ps["gemm"] * 1e6), "vote_subsets": round(fused_ps["vote"] * 1e6),
                   "fused_fallback": round(fused_ps["fallback"] * 1e6),
                   "_note": f"NEXT-3 capture ({R}_fused, N={CAPN['fused']}) scaled to N=1,000,000"},
      "per_sample": {k: round(v, 1) for k, v in per_sample.items()}}
json.dump(tj, open(f"{OUT}/traffic.json", "w"), indent=1)
print(json.dumps(tj, indent=1))
