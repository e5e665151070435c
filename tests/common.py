"""Shared test helpers: seeded synthetic inputs and oracle-built indexes."""
import functools
import hashlib

import numpy as np


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@functools.lru_cache(maxsize=None)
def index_case(n, d, blobs, n_clusters, k, seed=7, data_seed=42):
    """Data + oracle (C restatement) index: clusters, graph, PCA init."""
    from oracle import Oracle
    o = Oracle("port")
    x = o.gaussian_mixture(n, d, blobs, 10.0, data_seed)
    c = o.lsh_init(x, n_clusters, seed)
    c = o.kmeans_em(x, c, 100, o.default_kmeans_tol(x))
    g = o.build_knn(x, c, k)
    pca = o.pca_init(x, seed)
    return x, c, g, pca
