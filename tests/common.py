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


def manifold(n, d, seed=42, hidden=64, freq=4.0, noise=0.01):
    """A curved 2-D sheet in d dimensions: latent t ~ U[0,1]^2, features
    sin(t W1 + b) (hidden), linearly embedded, plus isotropic noise. Unlike
    isotropic blobs (NP@10 ~ 0.015 for the reference), its kNN
    neighbourhoods are 2-D, so a 2-D map can preserve them and NP@k
    discriminates between maps."""
    rng = np.random.default_rng(seed)
    t = rng.uniform(size=(n, 2))
    w1 = rng.normal(0.0, freq, (2, hidden))
    b = rng.uniform(0.0, 2 * np.pi, hidden)
    w2 = rng.normal(0.0, 1.0, (hidden, d)) / np.sqrt(hidden)
    x = np.sin(t @ w1 + b) @ w2 + noise * rng.normal(size=(n, d))
    return x.astype(np.float32), t
