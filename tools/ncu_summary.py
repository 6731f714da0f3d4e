#!/usr/bin/env python3
"""Summarizes ncu --set full reports (raw page + source-page stall totals)
into a JSON + markdown table for profiles/.

  python tools/ncu_summary.py gpurun_out/ncu_gaussian.ncu-rep [...] --out profiles/r1/ncu_summary
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "sm__maximum_warps_per_active_cycle_pct",
]
STALLS = ["stall_math", "stall_wait", "stall_not_selected", "stall_selected", "stall_short_sb", "stall_long_sb",
          "stall_barrier", "stall_mio", "stall_lg", "stall_branch_resolving", "stall_dispatch", "stall_no_inst",
          "stall_membar", "stall_drain", "stall_tex", "stall_sleep", "stall_misc"]


def ncu(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(out.stdout)))


def summarize(rep):
    rows = ncu(rep, "raw")
    if len(rows) < 3:
        return {"report": rep, "error": "no data"}
    head, units, vals = rows[0], rows[1], rows[2]
    res = {"report": rep, "kernel": vals[head.index("Kernel Name")] if "Kernel Name" in head else ""}
    for m in METRICS:
        if m in head:
            i = head.index(m)
            res[m] = f"{vals[i]} {units[i]}".strip()
    src = ncu(rep, "source", ["--print-source", "sass"])
    if len(src) > 2:
        h = src[1]
        tot = {}
        for r in src[2:]:
            for s in STALLS:
                if s in h:
                    try:
                        tot[s] = tot.get(s, 0) + int(r[h.index(s)] or 0)
                    except (ValueError, IndexError):
                        pass
        total = sum(tot.values()) or 1
        res["stall_share"] = {k: round(v / total, 3) for k, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+")
    ap.add_argument("--out", required=True)
    args = ap.parse_args()
    summ = [summarize(r) for r in args.reports]
    with open(args.out + ".json", "w") as f:
        json.dump(summ, f, indent=1)
    lines = ["| kernel | " + " | ".join(m.split(".")[0].replace("__", ".") for m in METRICS[:9]) + " | top stalls |",
             "|" + "---|" * 11]
    for s in summ:
        stalls = ", ".join(f"{k[6:]} {v:.0%}" for k, v in list(s.get("stall_share", {}).items())[:3])
        lines.append(f"| {s.get('kernel', '')[:40]} | " + " | ".join(s.get(m, "") for m in METRICS[:9]) +
                     f" | {stalls} |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
