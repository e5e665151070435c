"""Replay-mode epoch breakdown: wall time vs device time of the replay kernel.

    python tools/replay_probe.py [n] [clusters] [workers] [epochs] [graph]

graph: "synthetic" (random within-cluster lists, bench.synthetic_index) or
"knn" (the GPU index build on the device mixture: real kNN lists, whose
hub points lengthen the dependency chains)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2505_15511_b200 as nb  # noqa: E402

args = sys.argv[1:]
n, ncl, W, E = ([int(a) for a in args[:4]] + [1_000_000, 8, 8, 3][len(args[:4]):])[:4]
graph = args[4] if len(args) > 4 else "synthetic"
ctx = nb.Context(0)
if graph == "knn":
    x = nb.generate_mixture(n, 768, 64, 10.0, 42, ctx=ctx)
    cl = nb.kmeans_em_default_tol(x, nb.lsh_init(x, ncl, 7, ctx=ctx), 100, ctx=ctx)
    gk = nb.build_knn(x, cl, 15, mode="exact", ctx=ctx)
    del x
    torch.cuda.empty_cache()
    a, off, nbr = cl.assignment, gk.offsets, gk.neighbors
    init = np.random.default_rng(1234).standard_normal((n, 2))
    indeg = np.bincount(nbr, minlength=n)
    print(f"kNN in-degree: mean {indeg.mean():.1f} max {indeg.max()} (hub touches per epoch "
          f"~ in-degree + 1 + s)")
else:
    a, off, nbr, init = bench.synthetic_index(n, ncl, 15)
g = nb.KnnGraph(n, 15, off, nbr, np.zeros(0))
c = nb.ClusterAssignment(a, ncl, 16, np.zeros(0), np.zeros(0))
tr = nb.Trainer(g, c, init, nb.TrainConfig(epochs=200, workers=W, seed=7, sgd_mode="replay"), ctx=ctx)
tr.run(1)
s0, m0, e0 = tr.timing()
torch.cuda.synchronize()
t = time.perf_counter()
tr.run(E)
wall = (time.perf_counter() - t) / E
s1, m1, e1 = tr.timing()
print(f"n={n} C={ncl} W={W} graph={graph}: wall {wall*1e3:.1f} ms/epoch, replay kernel "
      f"{(s1-s0)/E:.1f} ms, means {(m1-m0)/E:.2f} ms, rest (draws, dependencies, host) "
      f"{wall*1e3-(s1-s0)/E-(m1-m0)/E:.1f} ms")
