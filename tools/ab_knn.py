"""A/B of the K <= 64 KNN kernels (collect-and-sort vs merge): config-3 microbench."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))

if __name__ == "__main__":
    import torch

    import bench_knn
    from paper_2304_07338_b200 import Context
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    with Context(0, stream=s.cuda_stream) as ctx:
        for mode in ("sel", "merge", "sel"):
            os.environ["PF_KNN_MERGE"] = "1" if mode == "merge" else "0"
            for K in (64, 32):
                r = bench_knn.run(ctx, K=K)
                print(mode, K, json.dumps({k: r[k] for k in ("queries_per_s", "ms_per_batch")}), flush=True)
