"""Summarise an ncu report (raw page) -> key metrics + warp stall breakdown.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_op_utcqmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    return [dict(zip(h, r)) for r in rows[2:]], dict(zip(h, units))


def main():
    path = sys.argv[1]
    recs, units = load(path)
    res = []
    for r in recs:
        d = {"kernel": r.get("Kernel Name", "")[:80]}
        for k in KEYS:
            if k in r:
                d[k] = r[k] + (" " + units.get(k, "") if units.get(k) else "")
        tensor = {k: r[k] for k in r if "tensor" in k and "pct" in k and r[k] not in ("0", "0.00", "")}
        d["tensor_pct"] = tensor
        pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
        stalls = {k[len(pre):-len(suf)]: float(r[k].replace(",", "")) for k in r
                  if k.startswith(pre) and k.endswith(suf) and r[k] not in ("", "n/a")}
        d["stalls_top"] = dict(sorted(stalls.items(), key=lambda kv: -float(kv[1]) if isinstance(kv[1], (int, float))
                                      else 0)[:10])
        res.append(d)
    txt = json.dumps(res, indent=1)
    print(txt)
    if "--json" in sys.argv:
        open(sys.argv[sys.argv.index("--json") + 1], "w").write(txt)


if __name__ == "__main__":
    main()
