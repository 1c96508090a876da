"""Refresh profiles/traffic.json (read by bench.py for roofline.traffic and the
issue figures) from ncu raw pages.  Tooling, not product.

usage: python tools/update_traffic.py <report.ncu-rep> [<report> ...]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parents[1] / "profiles" / "traffic.json"
KEYS = {
    "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed": "sm_issue_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "lanes",
    "gpu__time_duration.sum": "ncu_time",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1, "nsecond": 1e-6}


def main():
    doc = json.loads(OUT.read_text()) if OUT.exists() else {}
    kern = doc.get("kernels", {})
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").strip()
            d = {}
            for h, u, v in zip(hdr, units, r):
                if h in KEYS:
                    try:
                        d[KEYS[h]] = float(v.replace(",", "")) * SCALE.get(u, 1)
                    except ValueError:
                        pass
            e = {"dram_bytes": d.get("dram_read", 0) + d.get("dram_write", 0),
                 "sm_issue_active_pct": d.get("sm_issue_active_pct"), "fp64_pipe_pct": d.get("fp64_pipe_pct"),
                 "tensor_pipe_pct": d.get("tensor_pipe_pct"),
                 "lane_efficiency": d["lanes"] / 32 if "lanes" in d else None, "ncu_ms": d.get("ncu_time"),
                 "report": Path(rep).name}
            kern[name] = e
    doc = {"units": "per launch; ncu --set full --clock-control none (cold cache, serialised)",
           "source": "profiles/ (see README.md)", "kernels": kern}
    OUT.write_text(json.dumps(doc, indent=1) + "\n")
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
