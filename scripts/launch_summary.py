"""Summarise an ncu --metrics gpu__time_duration.sum,dram__bytes_* --csv launch list:
per kernel: launches, mean time, mean DRAM bytes; shares of our kernels' time.
    python scripts/launch_summary.py gpurun_out/launches.csv [--json out.json]
"""
import csv
import json
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr_i]
iid, ik, im, iv, iu = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
per = defaultdict(dict)
names = {}
for r in rows[hdr_i + 1:]:
    if len(r) <= iv:
        continue
    v = float(r[iv].replace(",", ""))
    u = r[iu]
    if u in ("usecond",):
        v *= 1e3
    elif u in ("msecond",):
        v *= 1e6
    elif u == "Kbyte":
        v *= 1e3
    elif u == "Mbyte":
        v *= 1e6
    elif u == "Gbyte":
        v *= 1e9
    per[r[iid]][r[im]] = v
    names[r[iid]] = r[ik]
agg = defaultdict(lambda: {"n": 0, "t_ns": 0.0, "rd": 0.0, "wr": 0.0})
for i, m in per.items():
    k = names[i]
    short = "arc_gemm_kernel" if "arc_gemm_kernel" in k else ("arc_quant_kernel" if "arc_quant_kernel" in k else k[:60])
    a = agg[short]
    a["n"] += 1
    a["t_ns"] += m.get("gpu__time_duration.sum", 0)
    a["rd"] += m.get("dram__bytes_read.sum", 0)
    a["wr"] += m.get("dram__bytes_write.sum", 0)
ours = {k: v for k, v in agg.items() if k.startswith("arc_")}
tot = sum(v["t_ns"] for v in ours.values())
out = {}
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]["t_ns"])[:12]:
    out[k] = {"launches": v["n"], "mean_us": v["t_ns"] / v["n"] / 1e3, "total_us": v["t_ns"] / 1e3,
              "mean_dram_bytes": (v["rd"] + v["wr"]) / v["n"],
              "share_of_arc_time": v["t_ns"] / tot if k in ours else None}
# the prefill step's launches (bench.py's timed region: 4 x (quant, GEMM) at M = 8192) vs the
# decode section's (M = 16): prefill GEMMs run > 40 us; each follows its site's quantize launch
pre = defaultdict(lambda: {"n": 0, "t_ns": 0.0, "bytes": 0.0})
ids = sorted(per, key=int)
for pos, i in enumerate(ids):
    k = names[i]
    t = per[i].get("gpu__time_duration.sum", 0)
    if not ("arc_gemm" in k and "reduce" not in k and t > 40e3):
        continue
    # a prefill GEMM and the quantize launch right before it (its site's activation)
    picks = [("arc_gemm_kernel", i)]
    if pos > 0 and "arc_quant_kernel" in names[ids[pos - 1]]:
        picks.append(("arc_quant_kernel", ids[pos - 1]))
    for key, j in picks:
        m = per[j]
        pre[key]["n"] += 1
        pre[key]["t_ns"] += m.get("gpu__time_duration.sum", 0)
        pre[key]["bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
ptot = sum(v["t_ns"] for v in pre.values())
out["prefill_step"] = {k: {"launches": v["n"], "mean_us": v["t_ns"] / max(v["n"], 1) / 1e3,
                           "mean_dram_bytes": v["bytes"] / max(v["n"], 1), "share_of_step": v["t_ns"] / ptot}
                       for k, v in pre.items()}
print(json.dumps(out, indent=1))
if "--json" in sys.argv:
    json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
