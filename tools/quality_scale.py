"""Final-map quality at scale (north star part 3) with the GPU metrics, which are
bit-identical to the reference's metric code: one GPU index, one GPU PCA init,
then the epoch loop in replay mode (the reference's exact trajectory) and in
throughput mode (hogwild) from the same start; NP@k on a row sample and random
triplet accuracy for both, plus wall times.

    python tools/quality_scale.py [n] [d] [blobs] [clusters] [epochs] [workers]
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2505_15511_b200 as nb  # noqa: E402


def main():
    a = [int(v) for v in sys.argv[1:]]
    n, d, blobs, C, E, W = (a + [1_000_000, 768, 64, 8, 100, 8][len(a):])[:6]
    ctx = nb.Context(0)
    out = {"n": n, "d": d, "blobs": blobs, "clusters": C, "epochs": E, "workers": W}
    t = time.perf_counter()
    x = nb.generate_mixture(n, d, blobs, 10.0, 42, ctx=ctx)
    c = nb.kmeans_em_default_tol(x, nb.lsh_init(x, C, 7, ctx=ctx), 100, ctx=ctx)
    g = nb.build_knn(x, c, 15, mode="bf16", ctx=ctx)
    torch.cuda.synchronize()
    out["index_s"] = round(time.perf_counter() - t, 2)
    t = time.perf_counter()
    init = nb.pca_init(x, 7, ctx=ctx, fast=True)
    out["pca_s"] = round(time.perf_counter() - t, 2)
    for mode in ("hogwild", "replay"):
        cfg = nb.TrainConfig(epochs=E, workers=W, seed=7, sgd_mode=mode)
        tr = nb.Trainer(g, c, init, cfg, ctx=ctx)
        t = time.perf_counter()
        losses = tr.run(E)
        torch.cuda.synchronize()
        secs = time.perf_counter() - t
        y = tr.layout()
        tr.close()
        t = time.perf_counter()
        npk, npse = nb.neighborhood_preservation(x, y, 10, 2000, 1, ctx=ctx)
        tri, trise = nb.random_triplet_accuracy(x, y, 200000, 1, ctx=ctx)
        out[mode] = {"train_s": round(secs, 2), "final_loss": float(losses[-1]),
                     "np10": npk, "np10_se": npse, "triplet": tri, "triplet_se": trise,
                     "metrics_s": round(time.perf_counter() - t, 2)}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
