"""Per-link latency of the replay dataflow kernel: every draw of a worker
touches its cluster's star centre (each row's list starts with it), so each
worker's epoch is ONE dependency chain of n / W draws; the replay kernel time
divided by n / W is the cost of one link (predecessor released -> observed ->
positions loaded -> draw computed -> stores released).

    python tools/replay_chain.py [n] [W] [epochs]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2505_15511_b200 as nb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 400_000
W = int(sys.argv[2]) if len(sys.argv) > 2 else 8
E = int(sys.argv[3]) if len(sys.argv) > 3 else 3
k, C = 15, W
rng = np.random.default_rng(3)
a = (np.arange(n) % C).astype(np.uint32)
centre = np.arange(C)  # first member of cluster c is point c
q = np.arange(n) // C
m = (n - a.astype(np.int64) + C - 1) // C
nb_ = np.empty((n, k), np.uint32)
nb_[:, 0] = centre[a]
for t in range(1, k):
    r = rng.integers(1, np.maximum(m, 2), dtype=np.int64)
    nb_[:, t] = (a + C * ((q + r) % m)).astype(np.uint32)
# the centre's own list: other members
nb_[:C, 0] = (np.arange(C) + C).astype(np.uint32)
off = (np.arange(n + 1, dtype=np.uint64) * k).astype(np.uint32)
ctx = nb.Context(0)
g = nb.KnnGraph(n, k, off, nb_.reshape(-1), np.zeros(0))
c = nb.ClusterAssignment(a, C, 16, np.zeros(0), np.zeros(0))
init = rng.standard_normal((n, 2))
tr = nb.Trainer(g, c, init, nb.TrainConfig(epochs=200, workers=W, seed=7, sgd_mode="replay", k=k),
                ctx=ctx)
tr.run(1)
s0, m0, e0 = tr.timing()
torch.cuda.synchronize()
tr.run(E)
s1, m1, e1 = tr.timing()
per = (s1 - s0) / E
print(f"n={n} W={W}: chain of {n // W} draws per worker, replay kernel {per:.1f} ms/epoch "
      f"-> {per * 1e3 / (n // W):.2f} us per link")
