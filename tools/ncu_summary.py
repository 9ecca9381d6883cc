"""Summarise ncu output for profiles/: (1) a launch list CSV (--metrics gpu__time_duration.sum) ->
per-kernel launches, total/avg time and share of the captured GPU time; (2) a --set full report
(.ncu-rep, read with `ncu -i ... --page raw --csv`) -> per-launch DRAM bytes, duration, achieved
bandwidth, registers, occupancy, FP64 pipe utilisation.

    python tools/ncu_summary.py launches gpurun_out/launches_cfg2.csv > profiles/...md
    python tools/ncu_summary.py full gpurun_out/prof.ncu-rep > profiles/...md
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict


def short(name: str) -> str:
    m = re.match(r"(?:void )?(?:hjb::)?([A-Za-z_0-9]+)(<[^()]*>)?", name)
    if not m:
        return name[:60]
    base = m.group(1) + (m.group(2) or "")
    if base.startswith("at") or "at::" in name[:40] or "elementwise" in name:
        return "torch:" + m.group(1)
    return base


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        ns = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)
        k = short(r[ki])
        agg[k][0] += 1
        agg[k][1] += ns
    tot = sum(v[1] for k, v in agg.items() if not k.startswith("torch:"))
    print(f"# ncu launch list: {path}\n")
    print(f"{sum(v[0] for v in agg.values())} launches captured; shares are of the libhjb kernels' summed "
          f"device time ({tot / 1e6:.2f} ms; cold-cache, serialised)\n")
    print("| kernel | launches | total ms | avg us | share |\n|---|---|---|---|---|")
    for k, (c, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if k.startswith("torch:"):
            continue
        print(f"| `{k}` | {c} | {ns / 1e6:.3f} | {ns / c / 1e3:.1f} | {ns / tot:.3f} |")


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
           "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
           "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"# ncu --set full summary: {path}\n")
    cols = [m for m in METRICS if m in hdr]
    print("| kernel | " + " | ".join(cols) + " |")
    print("|---|" + "---|" * len(cols))
    for r in rows[2:]:
        k = short(r[hdr.index("Kernel Name")])
        vals = []
        for m in cols:
            i = hdr.index(m)
            vals.append(f"{r[i]} {units[i]}".strip())
        print(f"| `{k}` | " + " | ".join(vals) + " |")


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
