#!/usr/bin/env python
"""Summarise an ncu --set full report and an ncu launch list into profiles/ (text + JSON).

    python tools/ncu_summary.py REPORT.ncu-rep LAUNCHES.csv OUT_PREFIX [events_per_launch_json]
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__bytes_write.sum.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__occupancy_limit_registers",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum",
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    report, launches, prefix = sys.argv[1:4]
    hdr, units, rows = raw(report)
    idx = {h: i for i, h in enumerate(hdr)}
    kernels = []
    for r in rows:
        k = {"kernel": r[idx["Kernel Name"]]}
        for m in METRICS:
            if m in idx:
                k[m] = f"{r[idx[m]]} {units[idx[m]]}".strip()
        stalls = [(hdr[i], float(r[i] or 0)) for i in range(len(hdr))
                  if hdr[i].startswith("smsp__average_warps_issue_stalled") and hdr[i].endswith("per_issue_active.ratio")]
        k["top_stalls_per_issue"] = {n.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""): v for n, v in sorted(stalls, key=lambda x: -x[1])[:6]}
        kernels.append(k)
    rows_l = [r for r in csv.reader(open(launches)) if len(r) > 10]
    h = rows_l[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows_l[1:]:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        name = r[ki].split("(")[0]
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    share = [{"kernel": k, "launches": cnt[k], "total_ms": v / 1e6, "share": v / s} for k, v in tot.most_common(12)]
    json.dump({"kernels": kernels, "launch_shares": share}, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu summary: {report}\n\n## Launch list shares ({launches})\n\n")
        f.write("| kernel | launches | total ms (cold, serialised) | share |\n|---|---|---|---|\n")
        for x in share:
            f.write(f"| `{x['kernel']}` | {x['launches']} | {x['total_ms']:.3f} | {x['share']:.3f} |\n")
        for k in kernels:
            f.write(f"\n## `{k['kernel']}`\n\n| metric | value |\n|---|---|\n")
            for m in METRICS:
                if m in k:
                    f.write(f"| {m} | {k[m]} |\n")
            f.write(f"| top stalls (per issue) | {k['top_stalls_per_issue']} |\n")
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    main()
