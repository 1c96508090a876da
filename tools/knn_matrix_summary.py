"""Compact one-line view of bench_knn.py JSON outputs (M queries/s per map / r_max). Tooling."""
import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, " ".join(f"{c['map'][:4]}/{c['r_max']}:{c['queries_per_s']/1e6:.0f}" for c in d["matrix"]))
    except Exception as e: print(f, "fail", e)
