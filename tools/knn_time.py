"""Warm kNN build timing: python tools/knn_time.py N D C MODE [BLOBS] (second of two builds)"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2505_15511_b200 as nb  # noqa: E402

n, d, C, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
blobs = int(sys.argv[5]) if len(sys.argv) > 5 else 64
ctx = nb.Context(0)
x = nb.generate_mixture(n, d, blobs, 10.0, 42, ctx=ctx)
c = nb.kmeans_em_default_tol(x, nb.lsh_init(x, C, 7, ctx=ctx), 100, ctx=ctx)
ts = []
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    nb.build_knn(x, c, 15, mode=mode, ctx=ctx)
    ts.append(time.perf_counter() - t)
print(f"{mode} n={n} C={C}: cold {ts[0]:.2f} s, warm {ts[1]:.2f} s, stats {ctx.knn_stats()} sub {ctx.knn_subcluster_rows()}")
