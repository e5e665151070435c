"""Quality parity on a structured dataset: throughput
(hogwild) fit vs the reference trajectory (replay fit, bit-identical to the
reference's fit) on the 2-D-sheet manifold of tests/common.py, NP@10 and
random-triplet accuracy by the GPU metrics (bit-identical to metrics.hpp).

    python tools/quality_manifold.py [n] [d] [epochs] [seeds] [workers] [noise]

(noise: per-feature noise of the sheet; at 1M rows the default 0.01 exceeds the
sheet's neighbour spacing, so the kNN graph is noise and NP@10 ~ 0.01 for any map)
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2505_15511_b200 as nb  # noqa: E402
from common import manifold  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 64
E = int(sys.argv[3]) if len(sys.argv) > 3 else 200
seeds = [int(s) for s in (sys.argv[4] if len(sys.argv) > 4 else "7,8,9").split(",")]
W = int(sys.argv[5]) if len(sys.argv) > 5 else 1
noise = float(sys.argv[6]) if len(sys.argv) > 6 else 0.01
ctx = nb.Context(0)
x, t = manifold(n, d, noise=noise)
sample = min(n, 5000)
for mode in ["replay", "hogwild"]:
    for s in seeds:
        t0 = time.time()
        lay = nb.fit(x, nb.TrainConfig(epochs=E, workers=W, seed=s, sgd_mode=mode), ctx=ctx)
        t1 = time.time()
        npv, npse = nb.neighborhood_preservation(x, lay, 10, sample=sample, seed=1, ctx=ctx)
        tr, trse = nb.random_triplet_accuracy(x, lay, 100000, 1, ctx=ctx)
        print(f"n={n} d={d} W={W} noise={noise:g} {mode:8s} seed {s}: NP@10 {npv:.4f} +- {npse:.4f}  "
              f"triplet {tr:.4f} +- {trse:.4f}  fit {t1 - t0:.1f} s", flush=True)
