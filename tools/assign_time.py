"""k-means timing at 10M x 768 (64 clusters) and 2M (16 clusters): lsh_init + kmeans_em wall
seconds, second of two runs. python tools/assign_time.py"""
import sys
import time
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2505_15511_b200 as nb  # noqa: E402
ctx = nb.Context(0)
for n, C in ((10_000_000, 64), (2_000_000, 16)):
    x = nb.generate_mixture(n, 768, 64, 10.0, 42, ctx=ctx)
    for _ in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        c0 = nb.lsh_init(x, C, 7, ctx=ctx)
        t1 = time.perf_counter()
        qe = []
        c = nb.kmeans_em_default_tol(x, c0, 100, qe_trace=qe, ctx=ctx)
        t2 = time.perf_counter()
    print(f"n={n} C={C}: lsh {t1 - t:.3f} s, kmeans {t2 - t1:.3f} s ({len(qe)} iterations)")
    del x
    torch.cuda.empty_cache()
