"""Time the GPU index build (lsh_init, kmeans_em default tol, build_knn) on
device-generated synthetic data: python tools/index_bench.py N D C [K]"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2505_15511_b200 as nb  # noqa: E402


def main():
    n, d, C = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    k = int(sys.argv[4]) if len(sys.argv) > 4 else 15
    ctx = nb.Context(0)
    t0 = time.perf_counter()
    x = nb.generate_mixture(n, d, 64, 10.0, 42, ctx=ctx)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    c0 = nb.lsh_init(x, C, 7, ctx=ctx)
    t2 = time.perf_counter()
    it = []
    c = nb.kmeans_em_default_tol(x, c0, 100, ctx=ctx)
    t3 = time.perf_counter()
    g = nb.build_knn(x, c, k, ctx=ctx)
    t4 = time.perf_counter()
    sizes = sorted(c.sizes.tolist())
    pairs = sum(s * s for s in c.sizes.tolist())
    print(json.dumps({"n": n, "d": d, "C": C, "k": k, "gen_s": t1 - t0, "lsh_s": t2 - t1,
                      "kmeans_s": t3 - t2, "knn_s": t4 - t3, "pairs": pairs,
                      "knn_pair_dims_per_s": pairs * d / (t4 - t3),
                      "knn_tflops_equiv": 2 * pairs * d / (t4 - t3) / 1e12,
                      "sizes_min_max": [sizes[0], sizes[-1]], "edges": int(g.offsets[-1])}))


if __name__ == "__main__":
    main()
