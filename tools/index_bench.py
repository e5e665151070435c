"""Time the GPU index build on device-generated synthetic data:
    python tools/index_bench.py N D C [--k 15] [--modes bf16,exact] [--recall]
Prints one JSON line: per-stage seconds, kNN TFLOP/s-equivalent (2 d sum s_r^2
per mode) and, with --recall, recall@k of bf16 against the exact graph."""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2505_15511_b200 as nb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("n", type=int)
    ap.add_argument("d", type=int)
    ap.add_argument("C", type=int)
    ap.add_argument("--k", type=int, default=15)
    ap.add_argument("--modes", default="bf16")
    ap.add_argument("--recall", action="store_true")
    a = ap.parse_args()
    ctx = nb.Context(0)
    t0 = time.perf_counter()
    x = nb.generate_mixture(a.n, a.d, 64, 10.0, 42, ctx=ctx)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    c0 = nb.lsh_init(x, a.C, 7, ctx=ctx)
    t2 = time.perf_counter()
    c = nb.kmeans_em_default_tol(x, c0, 100, ctx=ctx)
    t3 = time.perf_counter()
    pairs = int(sum(int(s) * int(s) for s in c.sizes))
    res = {"n": a.n, "d": a.d, "C": a.C, "k": a.k, "gen_s": t1 - t0, "lsh_s": t2 - t1,
           "kmeans_s": t3 - t2, "pairs": pairs,
           "sizes_min_max": [int(c.sizes.min()), int(c.sizes.max())]}
    graphs = {}
    for m in a.modes.split(","):
        torch.cuda.synchronize()
        s = time.perf_counter()
        graphs[m] = nb.build_knn(x, c, a.k, mode=m, ctx=ctx)
        e = time.perf_counter() - s
        res[f"knn_{m}_s"] = e
        res[f"knn_{m}_tc_uncertified_exhaustive"] = list(ctx.knn_stats())
        res[f"knn_{m}_subcluster_rows"] = ctx.knn_subcluster_rows()
        res[f"knn_{m}_tflops_equiv"] = 2 * pairs * a.d / e / 1e12
    if a.recall and "bf16" in graphs and "exact" in graphs:
        ge, gf = graphs["exact"], graphs["bf16"]
        k = a.k
        E = ge.neighbors.reshape(-1, k) if len(ge.neighbors) == a.n * k else None
        F = gf.neighbors.reshape(-1, k) if len(gf.neighbors) == a.n * k else None
        if E is not None and F is not None:
            hits = 0
            for lo in range(0, a.n, 200000):
                e_ = np.sort(E[lo:lo + 200000], axis=1)
                f_ = np.sort(F[lo:lo + 200000], axis=1)
                for j in range(k):  # count f_[:, j] in e_ rows
                    hits += int(np.sum(np.any(e_ == f_[:, j:j + 1], axis=1)))
            res["recall_at_k"] = hits / (a.n * k)
            res["exact_ids_equal_bf16"] = bool(np.array_equal(ge.neighbors, gf.neighbors))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
