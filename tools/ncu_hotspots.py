"""Per-source-line instruction / stall-sample shares of one kernel in an ncu
report (needs --import-source on and -lineinfo).  Tooling, not product.

usage: python tools/ncu_hotspots.py <report.ncu-rep> <kernel-regex> [top]
"""
import csv
import io
import subprocess
import sys


def hotspots(rep, kernel, top=20):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                          f"regex:{kernel}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "Line No"]
    if not hdr:
        return []
    res = []
    for r in rows[hdr[0] + 1:]:
        if r and r[0]:
            try:
                res.append((int(r[7]) if r[7] not in ("-", "") else 0, int(r[4]) if r[4] not in ("-", "") else 0,
                            r[0], r[1].strip()[:110]))
            except (ValueError, IndexError):
                pass
    ti = sum(x[0] for x in res) or 1
    ts = sum(x[1] for x in res) or 1
    res.sort(key=lambda x: -x[1])
    return [(line, i / ti, s / ts, src) for i, s, line, src in res[:top]]


if __name__ == "__main__":
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    print(f"# hotspots: {sys.argv[2]} in {sys.argv[1]}\n\n| line | inst share | stall share | source |\n|---|---|---|---|")
    for line, i, s, src in hotspots(sys.argv[1], sys.argv[2], top):
        print(f"| {line} | {i:.3f} | {s:.3f} | `{src.replace('|', '/')}` |")
