"""One kNN build on device data for profiling: python tools/knn_probe.py N D C MODE [BLOBS]
(BLOBS defaults to C: one Gaussian blob per cluster)"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2505_15511_b200 as nb  # noqa: E402

n, d, C, mode = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
ctx = nb.Context(0)
blobs = int(sys.argv[5]) if len(sys.argv) > 5 else C
x = nb.generate_mixture(n, d, blobs, 10.0, 42, ctx=ctx)
c = nb.kmeans_em_default_tol(x, nb.lsh_init(x, C, 7, ctx=ctx), 100, ctx=ctx)
torch.cuda.synchronize()
t = time.perf_counter()
g = nb.build_knn(x, c, 15, mode=mode, ctx=ctx)
print(mode, time.perf_counter() - t, "s", ctx.knn_stats())
