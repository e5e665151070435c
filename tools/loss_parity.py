"""Throughput (hogwild) vs deterministic (replay = the reference's trajectory)
per-epoch mean loss on the same GPU-built index and start layout:
    python tools/loss_parity.py [config] [epochs]      (config B or C)"""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2505_15511_b200 as nb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C"
E = int(sys.argv[2]) if len(sys.argv) > 2 else 20
n, d, blobs, C, W = bench.CONFIGS[name]
ctx = nb.Context(0)
x = nb.generate_mixture(n, d, blobs, 10.0, 42, ctx=ctx)
cl = nb.kmeans_em_default_tol(x, nb.lsh_init(x, C, 7, ctx=ctx), 100, ctx=ctx)
g = nb.build_knn(x, cl, 15, mode="exact", ctx=ctx)
del x
init = np.random.default_rng(1234).standard_normal((n, 2))
out = {}
for mode in ["replay", "hogwild"]:
    tr = nb.Trainer(g, cl, init, nb.TrainConfig(epochs=200, workers=W, seed=7, sgd_mode=mode),
                    ctx=ctx)
    out[mode] = tr.run(E)
print(f"config {name}: n={n} W={W}, {E} epochs from the same N(0,1) layout (lr schedule of 200 epochs)")
print("epoch   replay loss   hogwild loss   rel. diff")
for e in range(E):
    a, b = out["replay"][e], out["hogwild"][e]
    print(f"{e + 1:5d}  {a:12.6f}  {b:13.6f}  {(b - a) / a:+9.4f}")
