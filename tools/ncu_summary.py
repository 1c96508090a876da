"""Summarise an ncu report into profiles/ (markdown + JSON).  Tooling, not product.

usage: python tools/ncu_summary.py <report.ncu-rep> <out-stem> [--launches launches.csv]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__warps_eligible.avg.per_cycle_active", "sm__cycles_elapsed.avg.per_second",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            if h in KEYS or h in ("Kernel Name", "ID"):
                d[h] = {"value": v, "unit": u} if h in KEYS else v
        res.append(d)
    return res


def main():
    rep, stem = sys.argv[1], sys.argv[2]
    kernels = raw(rep)
    Path(stem).parent.mkdir(parents=True, exist_ok=True)
    Path(stem + ".json").write_text(json.dumps(kernels, indent=1))
    lines = [f"# ncu summary: {Path(rep).name}", ""]
    for k in kernels:
        lines.append(f"## {k.get('Kernel Name', '?')[:120]}")
        for key in KEYS:
            if key in k:
                lines.append(f"- `{key}`: {k[key]['value']} {k[key]['unit']}")
        lines.append("")
    Path(stem + ".md").write_text("\n".join(lines))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
