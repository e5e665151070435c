"""Wall time of lsh_init + kmeans_em_default_tol at config C (10M x 768, C = 64), twice."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2505_15511_b200 as nb
ctx = nb.Context(0)
x = nb.generate_mixture(10_000_000, 768, 64, 10.0, 42, ctx=ctx)
torch.cuda.synchronize()
for i in range(2):
    t = time.perf_counter(); c0 = nb.lsh_init(x, 64, 7, ctx=ctx); t1 = time.perf_counter()
    c = nb.kmeans_em_default_tol(x, c0, 100, ctx=ctx); t2 = time.perf_counter()
    print(f"lsh {t1-t:.3f} s  kmeans {t2-t1:.3f} s", flush=True)
