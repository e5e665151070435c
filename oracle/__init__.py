"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the two CPU checkers.

* ``Oracle("port")``      -> oracle/_build/libnomad_oracle.so, the plain-C
  restatement of the reference hot path (oracle/nomad_oracle.c).
* ``Oracle("reference")`` -> oracle/_ref/libnomad_ref.so, the unmodified
  reference headers (/root/reference/proj/include) compiled by
  oracle/Makefile with the pinned flags.

Both expose the same functions with the same argument meaning, so a test can
run either. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker /
baseline: the product (paper_2505_15511_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PATHS = {
    "port": os.path.join(HERE, "_build", "libnomad_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "libnomad_ref.so"),
}

KINDS = ["Io", "Dimension", "Validation", "Schema", "Parameter", "Config",
         "Degenerate", "Divergence", "Size", "Internal"]


class OracleError(RuntimeError):
    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind
        self.msg = msg


class TrainConfig(C.Structure):
    """Mirror of nomad::TrainConfig (optimizer.hpp:45-82) as a POD."""
    _fields_ = [("epochs", C.c_uint64), ("k", C.c_uint64), ("negatives", C.c_uint64),
                ("local_draws", C.c_uint64), ("batch_size", C.c_uint64),
                ("workers", C.c_uint64), ("n_clusters", C.c_uint64), ("seed", C.c_uint64),
                ("lr0", C.c_double), ("kmeans_max_iters", C.c_uint64),
                ("kmeans_tol", C.c_double), ("approx_all_but_own", C.c_int32),
                ("head_only", C.c_int32)]


def train_config(**kw) -> TrainConfig:
    d = dict(epochs=200, k=15, negatives=5, local_draws=5, batch_size=1024, workers=1,
             n_clusters=0, seed=0, lr0=0.0, kmeans_max_iters=100, kmeans_tol=-1.0,
             approx_all_but_own=0, head_only=0)
    d.update(kw)
    return TrainConfig(**d)


def build(quiet: bool = True) -> None:
    """Compile the checkers (make -C oracle). _ref only where /root/reference exists."""
    out = subprocess.run(["make", "-C", HERE], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout + out.stderr)


def available(which: str) -> bool:
    return os.path.exists(PATHS[which])


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t)) if a is not None else None


f32p, f64p, u32p, u64p = (C.POINTER(C.c_float), C.POINTER(C.c_double),
                          C.POINTER(C.c_uint32), C.POINTER(C.c_uint64))


@dataclass
class Clusters:
    assignment: np.ndarray  # u32[n]
    centroids: np.ndarray   # f64[C*d]
    sizes: np.ndarray       # u32[C]
    n_clusters: int
    dims: int


@dataclass
class Graph:
    offsets: np.ndarray     # u32[n+1]
    neighbors: np.ndarray   # u32[offsets[n]]
    distances: np.ndarray   # f64[offsets[n]]
    k: int


class Oracle:
    def __init__(self, which: str = "port"):
        self.which = which
        pre = "orc_" if which == "port" else "ref_"
        path = PATHS[which]
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        self.pre = pre
        L = self.lib
        def fn(name, res, args):
            f = getattr(L, pre + name)
            f.restype = res
            f.argtypes = args
            return f
        self._err = fn("last_error", C.c_char_p, [])
        self._stream_seed = fn("stream_seed", C.c_uint64, [C.c_uint64, C.c_uint64])
        self._rng_u64 = fn("rng_u64", None, [C.c_uint64, C.c_uint64, u64p])
        self._rng_gauss = fn("rng_gaussian", None, [C.c_uint64, C.c_uint64, f64p])
        self._rng_uidx = fn("rng_uniform_index", None, [C.c_uint64, C.c_uint64, C.c_uint64, u64p])
        self._irw = fn("inverse_rank_weights", C.c_int, [C.c_uint64, f64p])
        self._lr = fn("lr_schedule", C.c_double, [C.c_uint64, C.c_uint64, C.c_double])
        self._tol = fn("default_kmeans_tol", C.c_double, [f32p, C.c_uint64, C.c_uint64])
        self._lsh = fn("lsh_init", C.c_int, [f32p, C.c_uint64, C.c_uint64, C.c_uint64,
                                            C.c_uint64, u32p, f64p, u32p])
        self._km = fn("kmeans_em", C.c_int, [f32p, C.c_uint64, C.c_uint64, C.c_uint64, u32p,
                                            f64p, u32p, C.c_uint64, C.c_double, f64p, u64p])
        self._knn = fn("build_knn", C.c_int, [f32p, C.c_uint64, C.c_uint64, C.c_uint64, u32p,
                                             C.c_uint64, u32p, u32p, f64p])
        self._pca = fn("pca_init", C.c_int, [f32p, C.c_uint64, C.c_uint64, C.c_uint64, f64p])
        self._gm = fn("gather_means", C.c_int, [f64p, C.c_uint64, C.c_uint64, u32p, f64p])
        self._shard = fn("shard_clusters", C.c_int, [C.c_uint64, C.c_uint64, u32p, C.c_uint64,
                                                    u32p, u32p, u64p])
        self._grad = fn("nomad_gradient", C.c_int,
                        [f64p, C.c_uint64, C.c_uint32, u32p, f64p, C.c_uint64, u32p,
                         C.c_uint64, u32p, f64p, C.c_uint64, f64p, C.c_uint64, C.c_double,
                         C.c_uint64, f64p, f64p])
        self._knn_rows = fn("knn_rows", C.c_int, [f32p, u32p, C.c_uint64, C.c_uint64, u64p,
                                                 C.c_uint64, C.c_uint64, u32p, f64p, C.c_int32])
        self._nc_rows = fn("nearest_centroid_rows", None, [f32p, C.c_uint64, C.c_uint64, f64p,
                                                          C.c_uint64, u32p, C.c_int32])
        self._ccent = fn("cluster_centroid", None, [f32p, C.c_uint64, C.c_uint64, f64p])
        self._train = fn("train_epochs", C.c_int,
                         [C.c_uint64, C.c_uint64, u32p, u32p, u32p, C.c_uint64,
                          C.POINTER(TrainConfig), f64p, C.c_uint64, C.c_uint64, f64p, f64p,
                          C.c_int32, f64p])
        if which == "reference":
            self._fit = fn("fit", C.c_int, [f32p, C.c_uint64, C.c_uint64, C.POINTER(TrainConfig),
                                           f64p, u32p, u64p, u32p, u32p, f64p, f64p, f64p, f64p])
            self._np = fn("neighborhood_preservation", C.c_int,
                          [f32p, C.c_uint64, C.c_uint64, f64p, C.c_uint64, C.c_uint64,
                           C.c_uint64, f64p, f64p])
            self._tri = fn("random_triplet_accuracy", C.c_int,
                           [f32p, C.c_uint64, C.c_uint64, f64p, C.c_uint64, C.c_uint64, f64p,
                            f64p])
            self._npann = fn("neighborhood_preservation_ann", C.c_int,
                             [C.c_uint64, u32p, u32p, f64p, C.c_uint64, f64p])
            self._save = fn("save_layout", C.c_int, [C.c_char_p, f64p, C.c_uint64, C.c_void_p,
                                                     C.c_void_p])
            self._loadraw = fn("load_vectors_raw", C.c_int, [C.c_char_p, C.c_uint64, C.c_uint64,
                                                             C.c_void_p, u64p, u64p])
            self._qe = None
        else:
            self._fit = None
            self._qe = fn("quantization_error", C.c_double, [f32p, C.c_uint64, C.c_uint64, u32p, f64p])
            self._mix = fn("gaussian_mixture", None, [C.c_uint64, C.c_uint64, C.c_uint64,
                                                     C.c_double, C.c_uint64, f32p])

    # -- per-row checkers (row samples of configurations B-E) ------------
    def knn_rows(self, members: np.ndarray, ids: np.ndarray, queries, k: int,
                 threads: int = 0):
        """knn.hpp:88-106 for `queries` (indices into `members`, one cluster's
        rows in ascending id): (ids[nq, want], dists[nq, want])."""
        members = np.ascontiguousarray(members, np.float32)
        ids = np.ascontiguousarray(ids, np.uint32)
        q = np.ascontiguousarray(queries, np.uint64)
        m, d = members.shape
        oi = np.zeros((len(q), k), np.uint32)
        od = np.zeros((len(q), k), np.float64)
        want = self._knn_rows(_p(members, C.c_float), _p(ids, C.c_uint32), m, d,
                              _p(q, C.c_uint64), len(q), k, _p(oi, C.c_uint32),
                              _p(od, C.c_double), threads or (os.cpu_count() or 1))
        return oi[:, :want], od[:, :want]

    def nearest_centroid_rows(self, rows: np.ndarray, centroids: np.ndarray,
                              threads: int = 0) -> np.ndarray:
        """kmeans.hpp:56-68 per row."""
        rows = np.ascontiguousarray(rows, np.float32)
        cent = np.ascontiguousarray(centroids, np.float64).reshape(-1)
        nr, d = rows.shape
        out = np.zeros(nr, np.uint32)
        self._nc_rows(_p(rows, C.c_float), nr, d, _p(cent, C.c_double), len(cent) // d,
                      _p(out, C.c_uint32), threads or (os.cpu_count() or 1))
        return out

    def cluster_centroid(self, members: np.ndarray) -> np.ndarray:
        """kmeans.hpp:75-88 recompute_centroid from the member rows (ascending id)."""
        members = np.ascontiguousarray(members, np.float32)
        m, d = members.shape
        out = np.zeros(d, np.float64)
        self._ccent(_p(members, C.c_float), m, d, _p(out, C.c_double))
        return out

    # -- errors ---------------------------------------------------------
    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(KINDS[rc - 1], self._err().decode())

    # -- rng.hpp --------------------------------------------------------
    def stream_seed(self, base: int, stream: int) -> int:
        return int(self._stream_seed(base, stream))

    def rng_u64(self, seed: int, count: int) -> np.ndarray:
        out = np.zeros(count, np.uint64)
        self._rng_u64(seed, count, _p(out, C.c_uint64))
        return out

    def rng_gaussian(self, seed: int, count: int) -> np.ndarray:
        out = np.zeros(count, np.float64)
        self._rng_gauss(seed, count, _p(out, C.c_double))
        return out

    def rng_uniform_index(self, seed: int, bound: int, count: int) -> np.ndarray:
        out = np.zeros(count, np.uint64)
        self._rng_uidx(seed, bound, count, _p(out, C.c_uint64))
        return out

    # -- small tables -----------------------------------------------------
    def inverse_rank_weights(self, k: int) -> np.ndarray:
        out = np.zeros(max(k, 1), np.float64)
        self._check(self._irw(k, _p(out, C.c_double)))
        return out[:k]

    def lr_schedule(self, epoch: int, total: int, lr0: float) -> float:
        return float(self._lr(epoch, total, lr0))

    # -- index ------------------------------------------------------------
    def default_kmeans_tol(self, x: np.ndarray) -> float:
        x = np.ascontiguousarray(x, np.float32)
        return float(self._tol(_p(x, C.c_float), x.shape[0], x.shape[1]))

    def lsh_init(self, x: np.ndarray, n_clusters: int, seed: int) -> Clusters:
        x = np.ascontiguousarray(x, np.float32)
        n, d = x.shape
        a = np.zeros(n, np.uint32)
        c = np.zeros(n_clusters * d, np.float64)
        s = np.zeros(n_clusters, np.uint32)
        self._check(self._lsh(_p(x, C.c_float), n, d, n_clusters, seed, _p(a, C.c_uint32),
                              _p(c, C.c_double), _p(s, C.c_uint32)))
        return Clusters(a, c, s, n_clusters, d)

    def kmeans_em(self, x: np.ndarray, init: Clusters, max_iters: int = 100, tol: float = 0.0,
                  trace: bool = False):
        x = np.ascontiguousarray(x, np.float32)
        n, d = x.shape
        a, c, s = init.assignment.copy(), init.centroids.copy(), init.sizes.copy()
        qe = np.zeros(max(max_iters, 1), np.float64) if trace else None
        nt = np.zeros(1, np.uint64)
        self._check(self._km(_p(x, C.c_float), n, d, init.n_clusters, _p(a, C.c_uint32),
                             _p(c, C.c_double), _p(s, C.c_uint32), max_iters, tol,
                             _p(qe, C.c_double), _p(nt, C.c_uint64)))
        out = Clusters(a, c, s, init.n_clusters, d)
        return (out, qe[: int(nt[0])]) if trace else out

    def build_knn(self, x: np.ndarray, clusters: Clusters, k: int) -> Graph:
        x = np.ascontiguousarray(x, np.float32)
        n, d = x.shape
        off = np.zeros(n + 1, np.uint32)
        nb = np.zeros(max(n * k, 1), np.uint32)
        di = np.zeros(max(n * k, 1), np.float64)
        self._check(self._knn(_p(x, C.c_float), n, d, clusters.n_clusters,
                              _p(clusters.assignment, C.c_uint32), k, _p(off, C.c_uint32),
                              _p(nb, C.c_uint32), _p(di, C.c_double)))
        m = int(off[n])
        return Graph(off, nb[:m].copy(), di[:m].copy(), k)

    # -- layout -----------------------------------------------------------
    def pca_init(self, x: np.ndarray, seed: int = 0) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        n, d = x.shape
        out = np.zeros((n, 2), np.float64)
        self._check(self._pca(_p(x, C.c_float), n, d, seed, _p(out, C.c_double)))
        return out

    def gather_means(self, layout: np.ndarray, assignment: np.ndarray, n_clusters: int):
        layout = np.ascontiguousarray(layout, np.float64)
        assignment = np.ascontiguousarray(assignment, np.uint32)
        out = np.zeros((n_clusters, 2), np.float64)
        self._check(self._gm(_p(layout, C.c_double), layout.shape[0], n_clusters,
                             _p(assignment, C.c_uint32), _p(out, C.c_double)))
        return out

    def shard_clusters(self, assignment: np.ndarray, n_clusters: int, workers: int):
        assignment = np.ascontiguousarray(assignment, np.uint32)
        n = assignment.shape[0]
        c2w = np.zeros(n_clusters, np.uint32)
        wp = np.zeros(n, np.uint32)
        wo = np.zeros(workers + 1, np.uint64)
        self._check(self._shard(n, n_clusters, _p(assignment, C.c_uint32), workers,
                                _p(c2w, C.c_uint32), _p(wp, C.c_uint32), _p(wo, C.c_uint64)))
        return c2w, [wp[wo[w]:wo[w + 1]] for w in range(workers)]

    def nomad_gradient(self, layout, head, nbrs, weights, negs, remote, remote_probs, means,
                       local_mass, m_total):
        layout = np.ascontiguousarray(layout, np.float64)
        nbrs = np.ascontiguousarray(nbrs, np.uint32)
        weights = np.ascontiguousarray(weights, np.float64)
        negs = np.ascontiguousarray(negs, np.uint32)
        remote = np.ascontiguousarray(remote, np.uint32)
        remote_probs = np.ascontiguousarray(remote_probs, np.float64)
        means = np.ascontiguousarray(means, np.float64)
        g = np.zeros(2 * (1 + len(nbrs) + len(negs)), np.float64)
        loss = np.zeros(1, np.float64)
        self._check(self._grad(_p(layout, C.c_double), layout.shape[0], head,
                               _p(nbrs, C.c_uint32), _p(weights, C.c_double), len(nbrs),
                               _p(negs, C.c_uint32), len(negs), _p(remote, C.c_uint32),
                               _p(remote_probs, C.c_double), len(remote),
                               _p(means, C.c_double), means.shape[0], local_mass, m_total,
                               _p(loss, C.c_double), _p(g, C.c_double)))
        return float(loss[0]), g.reshape(-1, 2)

    def train_epochs(self, assignment, n_clusters, offsets, neighbors, k, cfg: TrainConfig,
                     layout, first_epoch=0, n_run=None, inline_workers=False):
        """Epoch loop of fit() from a given index; returns (layout, losses, means, seconds)."""
        assignment = np.ascontiguousarray(assignment, np.uint32)
        offsets = np.ascontiguousarray(offsets, np.uint32)
        neighbors = np.ascontiguousarray(neighbors, np.uint32)
        lay = np.ascontiguousarray(layout, np.float64).copy()
        n = assignment.shape[0]
        n_run = cfg.epochs - first_epoch if n_run is None else n_run
        losses = np.zeros(max(n_run, 1), np.float64)
        means = np.zeros((n_clusters, 2), np.float64)
        secs = np.zeros(1, np.float64)
        nb = neighbors if neighbors.size else np.zeros(1, np.uint32)
        self._check(self._train(n, n_clusters, _p(assignment, C.c_uint32),
                                _p(offsets, C.c_uint32), _p(nb, C.c_uint32), k,
                                C.byref(cfg), _p(lay, C.c_double), first_epoch, n_run,
                                _p(losses, C.c_double), _p(means, C.c_double),
                                1 if inline_workers else 0, _p(secs, C.c_double)))
        return lay, losses[:n_run], means, float(secs[0])

    def fit(self, x: np.ndarray, cfg: TrainConfig):
        """nomad::fit with the FitReport pieces (reference library only)."""
        if self._fit is None:
            raise RuntimeError("fit() is provided by the reference oracle only")
        x = np.ascontiguousarray(x, np.float32)
        n, d = x.shape
        k = cfg.k
        lay = np.zeros((n, 2), np.float64)
        a = np.zeros(n, np.uint32)
        nc = np.zeros(1, np.uint64)
        off = np.zeros(n + 1, np.uint32)
        nb = np.zeros(n * k, np.uint32)
        di = np.zeros(n * k, np.float64)
        pca = np.zeros((n, 2), np.float64)
        loss = np.zeros(max(cfg.epochs, 1), np.float64)
        means = np.zeros((n, 2), np.float64)  # upper bound on C
        self._check(self._fit(_p(x, C.c_float), n, d, C.byref(cfg), _p(lay, C.c_double),
                              _p(a, C.c_uint32), _p(nc, C.c_uint64), _p(off, C.c_uint32),
                              _p(nb, C.c_uint32), _p(di, C.c_double), _p(pca, C.c_double),
                              _p(loss, C.c_double), _p(means, C.c_double)))
        ncl = int(nc[0])
        m = int(off[n])
        return dict(layout=lay, assignment=a, n_clusters=ncl, offsets=off, neighbors=nb[:m],
                    distances=di[:m], pca=pca, epoch_loss=loss[: cfg.epochs],
                    final_means=means[:ncl])

    # -- reference-only quality metrics (metrics.hpp) -----------------------
    def neighborhood_preservation(self, x, layout, k=10, sample=0, seed=0):
        x = np.ascontiguousarray(x, np.float32)
        lay = np.ascontiguousarray(layout, np.float64)
        v, se = np.zeros(1), np.zeros(1)
        self._check(self._np(_p(x, C.c_float), x.shape[0], x.shape[1], _p(lay, C.c_double), k,
                             sample, seed, _p(v, C.c_double), _p(se, C.c_double)))
        return float(v[0]), float(se[0])

    def neighborhood_preservation_ann(self, offsets, neighbors, layout, k=10):
        """metrics.hpp:174-200 (reference library only)."""
        off = np.ascontiguousarray(offsets, np.uint32)
        nb = np.ascontiguousarray(neighbors, np.uint32)
        if nb.size == 0:
            nb = np.zeros(1, np.uint32)
        lay = np.ascontiguousarray(layout, np.float64)
        v = np.zeros(1)
        self._check(self._npann(len(off) - 1, _p(off, C.c_uint32), _p(nb, C.c_uint32),
                                _p(lay, C.c_double), k, _p(v, C.c_double)))
        return float(v[0])

    def save_layout(self, layout, path, ids=None, labels=None):
        """dataset.hpp:223-250 (reference library only)."""
        lay = np.ascontiguousarray(layout, np.float64)
        keep = []

        def arr(xs):
            if xs is None:
                return None
            bs = [str(v).encode() for v in xs]
            a = (C.c_char_p * len(bs))(*bs)
            keep.append((a, bs))
            return C.cast(a, C.c_void_p)
        self._check(self._save(path.encode(), _p(lay, C.c_double), lay.shape[0], arr(ids),
                               arr(labels)))

    def load_vectors_raw(self, path, rows=0, dims=0):
        """dataset.hpp:122-173 (reference library only) -> f32 array."""
        r, d = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
        self._check(self._loadraw(path.encode(), rows, dims, None, _p(r, C.c_uint64),
                                  _p(d, C.c_uint64)))
        out = np.empty((int(r[0]), int(d[0])), np.float32)
        self._check(self._loadraw(path.encode(), rows, dims, out.ctypes.data, _p(r, C.c_uint64),
                                  _p(d, C.c_uint64)))
        return out

    def random_triplet_accuracy(self, x, layout, count=100000, seed=0):
        x = np.ascontiguousarray(x, np.float32)
        lay = np.ascontiguousarray(layout, np.float64)
        v, se = np.zeros(1), np.zeros(1)
        self._check(self._tri(_p(x, C.c_float), x.shape[0], x.shape[1], _p(lay, C.c_double),
                              count, seed, _p(v, C.c_double), _p(se, C.c_double)))
        return float(v[0]), float(se[0])

    # -- port-only helpers --------------------------------------------------
    def quantization_error(self, x, clusters: Clusters) -> float:
        x = np.ascontiguousarray(x, np.float32)
        return float(self._qe(_p(x, C.c_float), x.shape[0], x.shape[1],
                              _p(clusters.assignment, C.c_uint32),
                              _p(clusters.centroids, C.c_double)))

    def gaussian_mixture(self, n: int, d: int, blobs: int, spread: float = 10.0,
                         seed: int = 42) -> np.ndarray:
        """Synthetic inputs of SURVEY §8(d): identical bytes on every box."""
        lib = self if self.which == "port" else Oracle("port")
        out = np.zeros((n, d), np.float32)
        lib._mix(n, d, blobs, spread, seed, _p(out, C.c_float))
        return out
