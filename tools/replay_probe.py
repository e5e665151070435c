"""Replay-mode epoch breakdown: wall time vs device time of the replay kernel.
python tools/replay_probe.py [n] [clusters] [workers] [epochs]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2505_15511_b200 as nb  # noqa: E402

n, ncl, W, E = ([int(a) for a in sys.argv[1:]] + [1_000_000, 8, 8, 3][len(sys.argv) - 1:])[:4]
a, off, nbr, init = bench.synthetic_index(n, ncl, 15)
ctx = nb.Context(0)
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
print(f"n={n} C={ncl} W={W}: wall {wall*1e3:.1f} ms/epoch, replay kernel {(s1-s0)/E:.1f} ms, "
      f"means {(m1-m0)/E:.2f} ms, host (tapes etc.) {wall*1e3-(s1-s0)/E-(m1-m0)/E:.1f} ms")
