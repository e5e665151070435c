"""Generate tests/golden/*.json from the REFERENCE itself (oracle/_ref, the
unmodified /root/reference headers compiled with the pinned flags).

Run here (where /root/reference exists):  python tests/make_golden.py
The fixtures hold SHA-256 digests of the reference's outputs (plus a few small
arrays as exact hex floats) on seeded synthetic inputs; tests/test_oracle.py
pins the C restatement against them and the GPU tests compare against both.
"""
import json
import os
import platform
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from common import sha  # noqa: E402
from oracle import Oracle, train_config  # noqa: E402

CASES = {
    # name: (n, d, blobs, clusters, k, workers, epochs_run, schedule)
    "small_w4": (3000, 32, 10, 8, 15, 4, 6, 10),
    "ragged_w4": (600, 8, 40, 40, 15, 4, 5, 5),
    "config_a_w1": (20000, 64, 10, 5, 15, 1, 3, 200),
    "config_a_w4": (20000, 64, 10, 5, 15, 4, 3, 200),
}


def hexs(a):
    return [float(v).hex() for v in np.asarray(a, np.float64).ravel()]


def main():
    R = Oracle("reference")
    out = {"generator": "tests/make_golden.py", "reference": "/root/reference/proj/include",
           "flags": "g++ -O2 -std=c++20 -ffp-contract=off",
           "gxx": subprocess.run(["g++", "--version"], capture_output=True, text=True).stdout.split("\n")[0],
           "glibc": platform.libc_ver()[1], "cases": {}}
    # rng / tables known answers
    out["rng"] = {
        "stream_seed_0_0": hex(R.stream_seed(0, 0)),
        "mt_u64_seed5_first8": [hex(int(v)) for v in R.rng_u64(5, 8)],
        "gaussian_seed5_sha_1001": sha(R.rng_gaussian(5, 1001)),
        "uniform_index_seed5_b77_sha_1000": sha(R.rng_uniform_index(5, 77, 1000)),
        "inverse_rank_weights_15": hexs(R.inverse_rank_weights(15)),
        "lr_9_of_10_lr0_100": float(R.lr_schedule(9, 10, 100.0)).hex(),
    }
    for name, (n, d, blobs, ncl, k, W, nrun, sched) in CASES.items():
        x = R.gaussian_mixture(n, d, blobs, 10.0, 42)
        c0 = R.lsh_init(x, ncl, 7)
        tol = R.default_kmeans_tol(x)
        c, qe = R.kmeans_em(x, c0, 100, tol, trace=True)
        g = R.build_knn(x, c, k)
        pca = R.pca_init(x, 7)
        cfg = train_config(epochs=sched, workers=W, seed=7)
        lay, loss, means, _ = R.train_epochs(c.assignment, ncl, g.offsets, g.neighbors, k, cfg,
                                             pca, 0, nrun)
        out["cases"][name] = dict(
            shape=[n, d, blobs, ncl, k, W, nrun, sched],
            data=sha(x), default_kmeans_tol=float(tol).hex(),
            lsh_assignment=sha(c0.assignment), lsh_centroids=sha(c0.centroids),
            lsh_sizes=c0.sizes.tolist(),
            km_assignment=sha(c.assignment), km_centroids=sha(c.centroids),
            km_sizes=c.sizes.tolist(), qe_trace=hexs(qe),
            knn_offsets=sha(g.offsets), knn_neighbors=sha(g.neighbors),
            knn_distances=sha(g.distances), pca=sha(pca),
            layout=sha(lay), epoch_loss=hexs(loss), final_means=sha(means))
        print(name, "done", flush=True)
    with open(os.path.join(HERE, "golden", "reference_goldens.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
