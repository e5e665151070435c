"""SGD kernel probe: per-epoch kernel time for variants of the throughput
epoch at config C (synthetic within-cluster graph):  python tools/sgd_probe.py"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_15511_b200 as nb  # noqa: E402


def main():
    n, d, blobs, ncl, W = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C"]
    a, off, nbr, init = bench.synthetic_index(n, ncl, 15)
    ctx = nb.Context(0)
    g = nb.KnnGraph(n, 15, off, nbr, np.zeros(0))
    c = nb.ClusterAssignment(a, ncl, d, np.zeros(0), np.zeros(0))
    out = {}
    for name, kw in [("hogwild", {}), ("head_only", {"head_only": True}),
                     ("all_but_own", {"approx": "non-own-cluster"}),
                     ("W1", {"workers": 1})]:
        cfg = nb.TrainConfig(epochs=200, workers=kw.pop("workers", W), seed=7,
                             sgd_mode="hogwild", **kw)
        tr = nb.Trainer(g, c, init, cfg, ctx=ctx)
        tr.run(3)
        s0, m0, e0 = tr.timing()
        tr.run(10)
        s1, m1, e1 = tr.timing()
        out[name] = {"sgd_ms": (s1 - s0) / 10, "means_ms": (m1 - m0) / 10}
        tr.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
