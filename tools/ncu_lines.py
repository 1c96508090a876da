"""Per-source-line warp instructions (per unit of work), lane occupancy and
stall share of one kernel from an ncu source-page CSV.  Tooling, not product.

usage: ncu -i rep --page source --csv --print-source cuda,sass -k regex:K > src.csv
       python tools/ncu_lines.py src.csv <units> [top]
"""
import csv
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    units = float(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    f, res = None, []
    for r in rows:
        if r and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) > 8 and r[0].isdigit() and not r[2].startswith("0x"):
            res.append((num(r[8]), num(r[7]), num(r[4]), f, r[0], r[1].strip()[:90]))
    tst = sum(x[2] for x in res) or 1
    ti = sum(x[1] for x in res)
    res.sort(key=lambda x: -x[1])
    print(f"warp instructions per unit: {ti / units:.2f}")
    for th, ins, st, f, line, src in res[:top]:
        print(f"{ins / units:7.3f} w/unit {th / max(ins, 1):5.1f} lanes  stall {st / tst:5.3f}  {f}:{line} {src}")


if __name__ == "__main__":
    main()
