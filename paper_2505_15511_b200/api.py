"""Host-side mirror of the reference library's API for the NOMAD hot path.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/nomad (cited per function), backed by
libnomad_b200.so. Arrays may be numpy arrays (host) or torch tensors (host or
CUDA); CUDA tensors are used in place.

    clusters = lsh_init(data, n_clusters, seed)              # kmeans.hpp:167
    clusters = kmeans_em(data, clusters, 100, tol)           # kmeans.hpp:257
    graph    = build_knn(data, clusters, k)                  # knn.hpp:65
    layout   = fit(data, TrainConfig(...), init_layout=pca)  # optimizer.hpp:327
    tr = Trainer(graph, clusters, init_layout, cfg); tr.run(E)   # epoch loop
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N
from ._native import NomadError, check, lib


# ---------------------------------------------------------------- arrays

def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _view(x, dtype):
    """(pointer, location, keepalive) of a contiguous array of dtype."""
    if _is_torch(x):
        import torch
        tdt = {np.float32: torch.float32, np.float64: torch.float64,
               np.uint32: torch.int32, np.int32: torch.int32}[dtype]
        if x.dtype != tdt and not (dtype == np.uint32 and x.dtype == torch.int32):
            x = x.to(tdt)
        x = x.contiguous()
        return x.data_ptr(), (N.DEVICE if x.is_cuda else N.HOST), x
    a = np.ascontiguousarray(x, dtype=dtype)
    return a.ctypes.data, N.HOST, a


def _dataset(data):
    """f32 rows, or bf16 rows when `data` is a torch.bfloat16 tensor (used in
    place; lsh_init, kmeans_em, build_knn(mode="bf16") and knn_recall)."""
    rows, dims = (int(data.shape[0]), int(data.shape[1]))
    if _is_torch(data):
        import torch
        if data.dtype == torch.bfloat16:
            x = data.contiguous()
            return (N.DatasetView(rows, dims, x.data_ptr(), N.DEVICE if x.is_cuda else N.HOST,
                                  N.BF16), x)
    p, loc, keep = _view(data, np.float32)
    return N.DatasetView(rows, dims, p, loc, N.F32), keep


# ---------------------------------------------------------------- types

@dataclass
class ClusterAssignment:
    """kmeans.hpp:32-43"""
    assignment: np.ndarray
    n_clusters: int
    dims: int
    centroids: np.ndarray
    sizes: np.ndarray

    def centroid(self, r: int) -> np.ndarray:
        return self.centroids[r * self.dims:(r + 1) * self.dims]

    def _view(self):
        self.assignment = np.ascontiguousarray(self.assignment, np.uint32)
        self.centroids = np.ascontiguousarray(self.centroids, np.float64).reshape(-1)
        self.sizes = np.ascontiguousarray(self.sizes, np.uint32)
        return N.ClustersView(len(self.assignment), self.n_clusters, self.dims,
                              self.assignment.ctypes.data, self.centroids.ctypes.data,
                              self.sizes.ctypes.data, N.HOST)


@dataclass
class KnnGraph:
    """knn.hpp:31-47 (CSR, squared distances)."""
    rows: int
    k: int
    offsets: np.ndarray
    neighbors: np.ndarray
    distances: np.ndarray

    def neighbor_count(self, i: int) -> int:
        return int(self.offsets[i + 1] - self.offsets[i])

    def neighbors_of(self, i: int) -> np.ndarray:
        return self.neighbors[self.offsets[i]:self.offsets[i + 1]]


@dataclass
class TrainConfig:
    """optimizer.hpp:45-82 plus engine-only fields (sgd_mode, knn_mode, hogwild_cap)."""
    epochs: int = 200
    k: int = 15
    negatives: int = 5
    local_draws: int = 5
    batch_size: int = 1024
    workers: int = 1
    n_clusters: int = 0
    seed: int = 0
    lr0: float = 0.0
    kmeans_max_iters: int = 100
    kmeans_tol: float = -1.0
    approx: str = "remote"          # "remote" | "non-own-cluster"
    head_only: bool = False
    verbose: bool = False
    sgd_mode: str = "replay"        # "replay" (bit-exact) | "hogwild" (throughput)
    knn_mode: str = "exact"         # "exact" | "bf16"
    hogwild_cap: int = 0
    hogwild_double_float: bool = False  # double-float position rows (1 RED.F32x2, 48-bit) instead of f64
    checkpoint_every: int = 0       # fit(): layout CSV every N epochs (optimizer.hpp:463-469)
    checkpoint_prefix: str = ""     # "<prefix>.epoch<N>.csv"

    def validate(self) -> None:  # optimizer.hpp:63-71
        if self.workers < 1:
            raise NomadError("Parameter", "workers must be >= 1")
        if self.k < 1:
            raise NomadError("Parameter", "k must be >= 1")
        if self.negatives < 1:
            raise NomadError("Parameter", "negatives must be >= 1")
        if self.local_draws < 1:
            raise NomadError("Parameter", "local draws must be >= 1")
        if self.batch_size < 1:
            raise NomadError("Parameter", "batch size must be >= 1")
        if self.n_clusters != 0 and self.n_clusters < self.workers:
            raise NomadError("Parameter", "clusters must be >= workers")

    def resolve_clusters(self, n: int) -> int:  # optimizer.hpp:73-77
        if self.n_clusters != 0:
            return min(self.n_clusters, n)
        return min(n, max((n + 4095) // 4096, self.workers, 2))

    def resolve_lr0(self, n: int) -> float:  # optimizer.hpp:79-81
        return self.lr0 if self.lr0 > 0.0 else n / 10.0

    def c_struct(self) -> N.TrainConfigC:
        return N.TrainConfigC(
            self.epochs, self.k, self.negatives, self.local_draws, self.batch_size,
            self.workers, self.n_clusters, self.seed & (2**64 - 1), float(self.lr0),
            self.kmeans_max_iters, float(self.kmeans_tol),
            1 if self.approx == "non-own-cluster" else 0, 1 if self.head_only else 0,
            self.checkpoint_every, self.checkpoint_prefix.encode() or None, None, None,
            {"replay": N.SGD_REPLAY, "hogwild": N.SGD_HOGWILD}[self.sgd_mode],
            {"exact": N.KNN_EXACT, "bf16": N.KNN_BF16, "exact_ffma": N.KNN_EXACT_FFMA}[self.knn_mode],
            self.hogwild_cap, 1 if self.hogwild_double_float else 0, 1 if self.verbose else 0)


# ---------------------------------------------------------------- context

class Context:
    """One CUDA device + stream; owns no data between calls."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        check(lib().nomad_b200_create(device, C.byref(h)))
        self.h = h

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def knn_stats(self):
        """(tc_uncertified_rows, exhaustive_rows) of this context's last build_knn."""
        a, b = C.c_uint64(), C.c_uint64()
        check(lib().nomad_b200_knn_stats(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def knn_subcluster_rows(self) -> int:
        """Rows of the last build_knn settled by the sub-cluster stage."""
        r = C.c_uint64()
        check(lib().nomad_b200_knn_subcluster_rows(self.h, C.byref(r)))
        return r.value

    def kernel_launches(self) -> int:
        return int(lib().nomad_b200_kernel_launches(self.h))

    def set_stream(self, stream_ptr: int | None) -> None:
        check(lib().nomad_b200_set_stream(self.h, stream_ptr))

    def close(self) -> None:
        if self.h and not getattr(self, "_borrowed", False):
            lib().nomad_b200_destroy(self.h)
        self.h = None


def _ctx(ctx: Optional[Context]) -> Context:
    return ctx if ctx is not None else Context.default()


class Group:
    """Several devices driven by this process (nomad_b200_group_create): the
    one-call form of the reference's W workers (optimizer.hpp:327-328,
    :399-408). Distinct devices are joined by NCCL (ncclCommInitAll); a
    repeated device ([0, 0, 0, 0]) runs G ranks on one GPU with a loopback
    exchange. Pass it to Trainer(..., group=g)."""

    def __init__(self, devices):
        devs = (C.c_int32 * len(devices))(*[int(d) for d in devices])
        h = C.c_void_p()
        check(lib().nomad_b200_group_create(C.cast(devs, C.c_void_p), len(devices), C.byref(h)))
        self.h = h
        self.devices = list(devices)
        self._live = 0          # trainers on this group; the contexts outlive them
        self._closing = False
        n, lb = C.c_int32(), C.c_int32()
        check(lib().nomad_b200_group_size(self.h, C.byref(n), C.byref(lb)))
        self.size, self.loopback = n.value, bool(lb.value)

    def context(self, rank: int = 0) -> "Context":
        """Rank r's context (owned by the group) for index builds etc."""
        h = C.c_void_p()
        check(lib().nomad_b200_group_context(self.h, rank, C.byref(h)))
        c = Context.__new__(Context)
        c.device, c.h, c._borrowed = self.devices[rank], h, True
        return c

    def close(self) -> None:
        """Destroys the contexts once no trainer uses them (garbage collection
        may finalise a trainer after its group)."""
        if getattr(self, "h", None):
            if self._live > 0:
                self._closing = True
                return
            lib().nomad_b200_group_destroy(self.h)
            self.h = None

    def _release(self) -> None:
        self._live -= 1
        if self._live == 0 and self._closing:
            self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- index

def default_kmeans_tol(data, ctx: Optional[Context] = None) -> float:
    """kmeans.hpp:157-161"""
    dv, keep = _dataset(data)
    out = C.c_double()
    check(lib().nomad_b200_default_kmeans_tol(_ctx(ctx).h, C.byref(dv), C.byref(out)))
    return out.value


def lsh_init(data, n_clusters: int, seed: int, ctx: Optional[Context] = None) -> ClusterAssignment:
    """kmeans.hpp:167-250"""
    dv, keep = _dataset(data)
    n, d = dv.rows, dv.dims
    ca = ClusterAssignment(np.zeros(n, np.uint32), int(n_clusters), d,
                           np.zeros(int(n_clusters) * d, np.float64),
                           np.zeros(int(n_clusters), np.uint32))
    v = ca._view()
    check(lib().nomad_b200_lsh_init(_ctx(ctx).h, C.byref(dv), n_clusters, seed & (2**64 - 1),
                                    C.byref(v)))
    return ca


def kmeans_em(data, init: ClusterAssignment, max_iters: int = 100, tol: float = 0.0,
              qe_trace: Optional[list] = None, ctx: Optional[Context] = None) -> ClusterAssignment:
    """kmeans.hpp:257-296 (init is taken by value, as the reference)."""
    dv, keep = _dataset(data)
    if len(init.assignment) != dv.rows or init.dims != dv.dims:
        raise NomadError("Parameter", "init assignment does not match dataset")
    ca = ClusterAssignment(np.array(init.assignment, np.uint32), init.n_clusters, init.dims,
                           np.array(init.centroids, np.float64).reshape(-1),
                           np.array(init.sizes, np.uint32))
    v = ca._view()
    trace = np.zeros(max(max_iters, 1), np.float64) if qe_trace is not None else None
    iters = C.c_uint64()
    check(lib().nomad_b200_kmeans_em(_ctx(ctx).h, C.byref(dv), C.byref(v), max_iters, tol,
                                     trace.ctypes.data if trace is not None else None,
                                     C.byref(iters)))
    if qe_trace is not None:
        qe_trace.clear()
        qe_trace.extend(trace[: iters.value].tolist())
    return ca


def kmeans_em_default_tol(data, init: ClusterAssignment, max_iters: int = 100,
                          qe_trace: Optional[list] = None,
                          ctx: Optional[Context] = None) -> ClusterAssignment:
    """kmeans_em(data, init, max_iters, default_kmeans_tol(data)) exactly as fit()
    calls it (optimizer.hpp:337-339), without the sequential tolerance sum
    unless a stop decision needs it."""
    dv, keep = _dataset(data)
    if len(init.assignment) != dv.rows or init.dims != dv.dims:
        raise NomadError("Parameter", "init assignment does not match dataset")
    ca = ClusterAssignment(np.array(init.assignment, np.uint32), init.n_clusters, init.dims,
                           np.array(init.centroids, np.float64).reshape(-1),
                           np.array(init.sizes, np.uint32))
    v = ca._view()
    trace = np.zeros(max(max_iters, 1), np.float64) if qe_trace is not None else None
    iters = C.c_uint64()
    check(lib().nomad_b200_kmeans_em_default_tol(_ctx(ctx).h, C.byref(dv), C.byref(v), max_iters,
                                                 trace.ctypes.data if trace is not None else None,
                                                 C.byref(iters)))
    if qe_trace is not None:
        qe_trace.clear()
        qe_trace.extend(trace[: iters.value].tolist())
    return ca


def build_knn(data, clusters: ClusterAssignment, k: int, mode: str = "exact",
              ctx: Optional[Context] = None, owned_clusters=None) -> KnnGraph:
    """knn.hpp:65-109. owned_clusters: build lists only for these clusters'
    rows (multi-GPU shards; other rows get empty lists)."""
    if k < 1:
        raise NomadError("Parameter", "k must be >= 1")
    dv, keep = _dataset(data)
    n = dv.rows
    v = clusters._view()
    off = np.zeros(n + 1, np.uint32)
    nb = np.zeros(max(n * k, 1), np.uint32)
    di = np.zeros(max(n * k, 1), np.float64)
    gv = N.GraphView(n, k, off.ctypes.data, nb.ctypes.data, di.ctypes.data, N.HOST)
    km = {"exact": N.KNN_EXACT, "bf16": N.KNN_BF16, "exact_ffma": N.KNN_EXACT_FFMA}[mode]
    if owned_clusters is None:
        check(lib().nomad_b200_build_knn(_ctx(ctx).h, C.byref(dv), C.byref(v), k, km, C.byref(gv)))
    else:
        oc = np.ascontiguousarray(owned_clusters, np.uint32)
        check(lib().nomad_b200_build_knn_shard(_ctx(ctx).h, C.byref(dv), C.byref(v), k, km,
                                               len(oc), oc.ctypes.data if len(oc) else None,
                                               C.byref(gv)))
    m = int(off[n])
    return KnnGraph(n, k, off, nb[:m], di[:m])


def knn_recall(data, clusters: ClusterAssignment, graph: KnnGraph, sample: int = 20000,
               seed: int = 0, ctx: Optional[Context] = None) -> float:
    """recall@k of `graph` vs exact lists recomputed in fp64 for `sample` rows."""
    dv, keep = _dataset(data)
    cv = clusters._view()
    off = np.ascontiguousarray(graph.offsets, np.uint32)
    nb_ = np.ascontiguousarray(graph.neighbors, np.uint32)
    if nb_.size == 0:
        nb_ = np.zeros(1, np.uint32)
    gv = N.GraphView(graph.rows, graph.k, off.ctypes.data, nb_.ctypes.data, None, N.HOST)
    out = C.c_double()
    check(lib().nomad_b200_knn_recall(_ctx(ctx).h, C.byref(dv), C.byref(cv), C.byref(gv), sample,
                                      seed, C.byref(out)))
    return out.value


# ---------------------------------------------------------------- data I/O

def load_vectors_raw(path: str, rows: int = 0, dims: int = 0, device: bool = False,
                     ctx: Optional[Context] = None):
    """dataset.hpp:122-173 (raw little-endian f32). device=True streams the file
    into a CUDA float32 tensor through pinned buffers; else a numpy array."""
    r, d = C.c_uint64(), C.c_uint64()
    h = _ctx(ctx).h if device else None
    check(lib().nomad_b200_load_vectors_raw(h, path.encode(), rows, dims, None, N.HOST,
                                            C.byref(r), C.byref(d)))
    if device:
        import torch
        out = torch.empty((r.value, d.value), dtype=torch.float32, device=f"cuda:{_ctx(ctx).device}")
        check(lib().nomad_b200_load_vectors_raw(h, path.encode(), rows, dims, out.data_ptr(),
                                                N.DEVICE, None, None))
        return out
    out = np.empty((r.value, d.value), np.float32)
    check(lib().nomad_b200_load_vectors_raw(None, path.encode(), rows, dims, out.ctypes.data,
                                            N.HOST, None, None))
    return out


def _str_array(xs):
    if xs is None:
        return None, None
    bs = [str(v).encode() for v in xs]
    arr = (C.c_char_p * len(bs))(*bs)
    return C.cast(arr, C.c_void_p), (arr, bs)


def save_layout(layout, path: str, ids=None, labels=None) -> None:
    """dataset.hpp:223-250: `id,x,y[,label]` CSV with %.17g (byte-identical)."""
    lay = np.ascontiguousarray(layout, np.float64).reshape(-1, 2)
    ip, ik = _str_array(ids)
    lp, lk = _str_array(labels)
    check(lib().nomad_b200_save_layout_csv(path.encode(), lay.ctypes.data, lay.shape[0], ip, lp))


def save_layout_f64(layout, path: str) -> None:
    """Raw little-endian f64 rows x 2."""
    lay = np.ascontiguousarray(layout, np.float64).reshape(-1, 2)
    check(lib().nomad_b200_save_layout_f64(path.encode(), lay.ctypes.data, lay.shape[0]))


# ---------------------------------------------------------------- quality metrics

def neighborhood_preservation(data, layout, k: int = 10, sample: int = 0, seed: int = 0,
                              ctx: Optional[Context] = None):
    """metrics.hpp:113-168 on the GPU -> (value, std_error), bit-identical to the
    reference's (same sampled rows, exact high-d and 2-D neighbours)."""
    dv, keep = _dataset(data)
    lp, lloc, lkeep = _view(layout, np.float64)
    v, se = C.c_double(), C.c_double()
    check(lib().nomad_b200_neighborhood_preservation(_ctx(ctx).h, C.byref(dv), lp, lloc, k, sample,
                                                     seed & (2**64 - 1), C.byref(v), C.byref(se)))
    return v.value, se.value


def neighborhood_preservation_ann(graph: KnnGraph, layout, k: int = 10,
                                  ctx: Optional[Context] = None) -> float:
    """metrics.hpp:174-200 on the GPU (graph neighbourhoods vs exact 2-D), bit-identical."""
    off = np.ascontiguousarray(graph.offsets, np.uint32)
    nb_ = np.ascontiguousarray(graph.neighbors, np.uint32)
    if nb_.size == 0:
        nb_ = np.zeros(1, np.uint32)
    gv = N.GraphView(graph.rows, graph.k, off.ctypes.data, nb_.ctypes.data, None, N.HOST)
    lp, lloc, lkeep = _view(layout, np.float64)
    v = C.c_double()
    check(lib().nomad_b200_neighborhood_preservation_ann(_ctx(ctx).h, C.byref(gv), lp, lloc, k,
                                                         C.byref(v)))
    return v.value


def random_triplet_accuracy(data, layout, count: int = 100000, seed: int = 0,
                            ctx: Optional[Context] = None):
    """metrics.hpp:205-243 on the GPU -> (value, std_error), bit-identical."""
    dv, keep = _dataset(data)
    lp, lloc, lkeep = _view(layout, np.float64)
    v, se = C.c_double(), C.c_double()
    check(lib().nomad_b200_random_triplet_accuracy(_ctx(ctx).h, C.byref(dv), lp, lloc, count,
                                                   seed & (2**64 - 1), C.byref(v), C.byref(se)))
    return v.value, se.value


# ---------------------------------------------------------------- training

@dataclass
class CommLog:
    """optimizer.hpp:178-189 totals."""
    epochs: int
    messages: int
    payload_doubles: int
    payload_counts: int


class Trainer:
    """The epoch loop of fit() (optimizer.hpp:342-470) on the GPU.

    graph: KnnGraph (or a dict of device tensors offsets/neighbors), clusters:
    ClusterAssignment (assignment + n_clusters), init_layout: n x 2 f64.
    Multi-GPU: rank/world_size and a 128-byte NCCL unique id (one process
    per GPU), or group=Group([...]) (one process drives every rank).
    """

    def __init__(self, graph, clusters, init_layout, cfg: TrainConfig, rank: int = 0,
                 world_size: int = 1, nccl_id: Optional[bytes] = None,
                 ctx: Optional[Context] = None, group: Optional[Group] = None):
        cfg.validate()
        self.group = group
        self.ctx = group.context(0) if group is not None else _ctx(ctx)
        self.cfg = cfg
        if isinstance(graph, KnnGraph):
            n, k = graph.rows, graph.k
            offs, nbrs = graph.offsets, graph.neighbors
        else:
            n, k = int(graph["rows"]), int(graph["k"])
            offs, nbrs = graph["offsets"], graph["neighbors"]
        po, lo, ko = _view(offs, np.uint32)
        nbrs_nonempty = nbrs if len(nbrs) else np.zeros(1, np.uint32)
        pn, ln, kn = _view(nbrs_nonempty, np.uint32)
        if lo != ln:
            raise NomadError("Parameter", "graph offsets/neighbors must share a location")
        gv = N.GraphView(n, k, po, pn, None, lo)
        if isinstance(clusters, ClusterAssignment):
            asg, ncl = clusters.assignment, clusters.n_clusters
        else:
            asg, ncl = clusters["assignment"], int(clusters["n_clusters"])
        pa, la, ka = _view(asg, np.uint32)
        cv = N.ClustersView(n, ncl, 0, pa, None, None, la)
        pl, ll, kl = _view(init_layout, np.float64)
        self.n, self.n_clusters = n, ncl
        self._keep = (ko, kn, ka, kl)
        c = cfg.c_struct()
        idbuf = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        h = C.c_void_p()
        if group is not None:
            check(lib().nomad_b200_group_trainer_create(group.h, C.byref(gv), C.byref(cv), pl, ll,
                                                        C.byref(c), C.byref(h)))
        else:
            check(lib().nomad_b200_trainer_create(self.ctx.h, C.byref(gv), C.byref(cv), pl, ll,
                                                  C.byref(c), rank, world_size, idbuf, C.byref(h)))
        self.h = h
        r = C.c_int32()
        check(lib().nomad_b200_trainer_ranks(self.h, C.byref(r)))
        self.ranks = r.value
        if group is not None:
            group._live += 1

    def run(self, n_epochs: int) -> np.ndarray:
        out = np.zeros(max(n_epochs, 1), np.float64)
        check(lib().nomad_b200_trainer_run(self.h, n_epochs, out.ctypes.data))
        return out[:n_epochs]

    def layout(self, out=None) -> np.ndarray:
        if out is not None and _is_torch(out) and out.is_cuda:
            check(lib().nomad_b200_trainer_layout(self.h, out.data_ptr(), N.DEVICE))
            return out
        arr = np.zeros((self.n, 2), np.float64) if out is None else out
        check(lib().nomad_b200_trainer_layout(self.h, arr.ctypes.data, N.HOST))
        return arr

    def means(self):
        m = np.zeros((self.n_clusters, 2), np.float64)
        c = np.zeros(self.n_clusters, np.uint32)
        check(lib().nomad_b200_trainer_means(self.h, m.ctypes.data, c.ctypes.data))
        return m, c

    def comm_log(self) -> CommLog:
        v = [C.c_uint64() for _ in range(4)]
        check(lib().nomad_b200_trainer_comm(self.h, *[C.byref(x) for x in v]))
        return CommLog(*[x.value for x in v])

    def set_layout(self, layout) -> None:
        p, loc, keep = _view(layout, np.float64)
        check(lib().nomad_b200_trainer_set_layout(self.h, p, loc))

    def timing(self):
        """(sgd_ms, means_ms, epochs): device time accumulated over all epochs run."""
        a, b, e = C.c_double(), C.c_double(), C.c_uint64()
        check(lib().nomad_b200_trainer_timing(self.h, C.byref(a), C.byref(b), C.byref(e)))
        return a.value, b.value, e.value

    def seek(self, epoch: int) -> None:
        """Continue the schedule at `epoch` (resume after set_layout(checkpoint))."""
        check(lib().nomad_b200_trainer_seek(self.h, epoch))

    def progress(self):
        e, u = C.c_uint64(), C.c_uint64()
        check(lib().nomad_b200_trainer_progress(self.h, C.byref(e), C.byref(u)))
        return e.value, u.value

    def close(self):
        if getattr(self, "h", None):
            lib().nomad_b200_trainer_destroy(self.h)
            self.h = None
            if getattr(self, "group", None) is not None:
                self.group._release()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ConditionalAffinity:
    """affinity.hpp:47-63: inverse-rank p(j|i) per edge (CSR as the graph)."""
    rows: int
    offsets: np.ndarray
    neighbors: np.ndarray
    weights: np.ndarray
    eligible_heads: np.ndarray


@dataclass
class ShardPlan:
    """optimizer.hpp:94-100."""
    workers: int
    cluster_to_worker: np.ndarray
    worker_clusters: list
    worker_points: list


@dataclass
class FitReport:
    """optimizer.hpp:312-321, every field from the engine's outputs."""
    clusters: Optional[ClusterAssignment] = None
    graph: Optional[KnnGraph] = None
    affinity: Optional[ConditionalAffinity] = None
    plan: Optional[ShardPlan] = None
    pca: Optional[np.ndarray] = None
    final_means: Optional[np.ndarray] = None
    comm: Optional[CommLog] = None
    epoch_mean_loss: list = field(default_factory=list)


def fit(data, config: TrainConfig, init_layout=None, report: Optional[FitReport] = None,
        ctx: Optional[Context] = None, group: Optional[Group] = None) -> np.ndarray:
    """optimizer.hpp:327-482. init_layout: the PCA initialisation (n x 2; None:
    the GPU PCA). group: run the epochs on every rank of a Group."""
    config.validate()
    dv, keep = _dataset(data)
    n, d = dv.rows, dv.dims
    ncl = config.resolve_clusters(n)
    k = config.k
    out = np.zeros((n, 2), np.float64)
    pl = None
    if init_layout is not None:
        il = np.ascontiguousarray(init_layout, np.float64)
        pl = il.ctypes.data
    c = config.c_struct()
    rep = N.FitReportC()
    hold = []
    if report is not None:  # full outputs only when asked for (12 n k bytes of graph)
        ca = ClusterAssignment(np.zeros(n, np.uint32), ncl, d, np.zeros(ncl * d, np.float64),
                               np.zeros(ncl, np.uint32))
        cv = ca._view()
        off = np.zeros(n + 1, np.uint32)
        nb = np.zeros(max(n * k, 1), np.uint32)
        di = np.zeros(max(n * k, 1), np.float64)
        gv = N.GraphView(n, k, off.ctypes.data, nb.ctypes.data, di.ctypes.data, N.HOST)
        losses = np.zeros(max(config.epochs, 1), np.float64)
        pca = np.zeros((n, 2), np.float64)
        means = np.zeros((ncl, 2), np.float64)
        c2w = np.zeros(ncl, np.uint32)
        aw = np.zeros(max(n * k, 1), np.float64)
        el = np.zeros(max(n, 1), np.uint32)
        hold = [cv, gv]
        rep.clusters, rep.graph = C.addressof(cv), C.addressof(gv)
        rep.epoch_mean_loss, rep.pca = losses.ctypes.data, pca.ctypes.data
        rep.final_means, rep.cluster_to_worker = means.ctypes.data, c2w.ctypes.data
        rep.affinity_weights, rep.eligible_heads = aw.ctypes.data, el.ctypes.data
    h = group.h if group is not None else _ctx(ctx).h
    check(lib().nomad_b200_fit_ex(None if group is not None else h,
                                  h if group is not None else None, C.byref(dv), C.byref(c), pl,
                                  out.ctypes.data, C.byref(rep)))
    del hold
    if report is not None:
        m = int(off[n])
        report.clusters = ca
        report.graph = KnnGraph(n, k, off, nb[:m], di[:m])
        report.affinity = ConditionalAffinity(n, off, nb[:m], aw[:m], el[:rep.n_eligible])
        a = ca.assignment
        report.plan = ShardPlan(config.workers, c2w,
                                [np.nonzero(c2w == w)[0].astype(np.uint32)
                                 for w in range(config.workers)],
                                [np.nonzero(c2w[a] == w)[0].astype(np.uint32)
                                 for w in range(config.workers)])
        report.pca = pca
        report.final_means = means
        report.comm = CommLog(rep.comm_epochs, rep.comm_messages, rep.comm_payload_doubles,
                              rep.comm_payload_counts)
        report.epoch_mean_loss = losses[: config.epochs].tolist()
    return out


def pca_init(data, seed: int = 0, ctx: Optional[Context] = None, fast: bool = False) -> np.ndarray:
    """pca.hpp:79-218 on the GPU: bit-identical (default) or, fast=True, with the
    covariance formed once (tolerance parity, ~2 data passes)."""
    dv, keep = _dataset(data)
    out = np.zeros((dv.rows, 2), np.float64)
    fn = lib().nomad_b200_pca_init_fast if fast else lib().nomad_b200_pca_init
    check(fn(_ctx(ctx).h, C.byref(dv), seed & (2**64 - 1), out.ctypes.data, N.HOST))
    return out


def generate_mixture(rows: int, dims: int, blobs: int, spread: float = 10.0, seed: int = 42,
                     out=None, ctx: Optional[Context] = None, dtype: str = "f32"):
    """Device synthetic Gaussian mixture into a CUDA tensor (rows x dims);
    dtype "bf16": the same values rounded to bfloat16 (the 60M configuration)."""
    import torch
    cx = _ctx(ctx)
    bf = dtype == "bf16"
    if dtype not in ("f32", "bf16"):
        raise NomadError("Parameter", "dtype must be 'f32' or 'bf16'")
    if out is None:
        out = torch.empty((rows, dims), dtype=torch.bfloat16 if bf else torch.float32,
                          device=f"cuda:{cx.device}")
    fn = lib().nomad_b200_generate_mixture_bf16 if bf else lib().nomad_b200_generate_mixture
    check(fn(cx.h, rows, dims, blobs, spread, seed, out.data_ptr()))
    return out


def generate_mixture_rows(row0: int, rows: int, dims: int, blobs: int, spread: float = 10.0,
                          seed: int = 42, ctx: Optional[Context] = None, dtype: str = "f32"):
    """Rows [row0, row0 + rows) of generate_mixture's matrix (a rank's share)."""
    import torch
    cx = _ctx(ctx)
    bf = dtype == "bf16"
    out = torch.empty((rows, dims), dtype=torch.bfloat16 if bf else torch.float32,
                      device=f"cuda:{cx.device}")
    check(lib().nomad_b200_generate_mixture_rows(cx.h, row0, rows, dims, blobs, spread, seed,
                                                 N.BF16 if bf else N.F32, out.data_ptr()))
    return out


def _sharded_outputs(n_total, C, d, k):
    ca = ClusterAssignment(np.zeros(n_total, np.uint32), C, d, np.zeros(C * d, np.float64),
                           np.zeros(C, np.uint32))
    off = np.zeros(n_total + 1, np.uint32)
    nb = np.zeros(max(n_total * k, 1), np.uint32)
    di = np.zeros(max(n_total * k, 1), np.float64)
    return ca, off, nb, di


def index_sharded(rows, row0: int, n_total: int, n_clusters: int, seed: int, workers: int,
                  k: int = 15, knn_mode: str = "exact", rank: int = 0, world_size: int = 1,
                  nccl_id: Optional[bytes] = None, max_iters: int = 100, tol: float = -1.0,
                  ctx: Optional[Context] = None):
    """Row-sharded lsh_init + kmeans_em + build_knn for one rank of a
    multi-process run (nomad_b200_index_sharded): this rank holds rows
    [row0, row0 + len(rows)). Returns (ClusterAssignment over all n_total
    rows, KnnGraph holding this rank's clusters' lists)."""
    dv, keep = _dataset(rows)
    C_, d = int(n_clusters), dv.dims
    ca, off, nb, di = _sharded_outputs(n_total, C_, d, k)
    cv = ca._view()
    gv = N.GraphView(n_total, k, off.ctypes.data, nb.ctypes.data, di.ctypes.data, N.HOST)
    idbuf = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
    km = {"exact": N.KNN_EXACT, "bf16": N.KNN_BF16, "exact_ffma": N.KNN_EXACT_FFMA}[knn_mode]
    check(lib().nomad_b200_index_sharded(_ctx(ctx).h, rank, world_size, idbuf, C.byref(dv), row0,
                                         n_total, C_, seed & (2**64 - 1), max_iters, tol, workers,
                                         k, km, C.byref(cv), C.byref(gv)))
    m = int(off[n_total])
    return ca, KnnGraph(n_total, k, off, nb[:m], di[:m])


def group_index_sharded(group: "Group", rows: list, row0: list, n_total: int, n_clusters: int,
                        seed: int, workers: int, k: int = 15, knn_mode: str = "exact",
                        max_iters: int = 100, tol: float = -1.0):
    """The row-sharded index build over the ranks of a Group (rows[r] on rank
    r's device): (ClusterAssignment, KnnGraph with every rank's lists)."""
    views, keeps = [], []
    for r in rows:
        v, kp = _dataset(r)
        views.append(v)
        keeps.append(kp)
    arr = (N.DatasetView * len(views))(*views)
    r0 = np.ascontiguousarray(row0, np.uint64)
    C_, d = int(n_clusters), views[0].dims
    ca, off, nb, di = _sharded_outputs(n_total, C_, d, k)
    cv = ca._view()
    gv = N.GraphView(n_total, k, off.ctypes.data, nb.ctypes.data, di.ctypes.data, N.HOST)
    km = {"exact": N.KNN_EXACT, "bf16": N.KNN_BF16, "exact_ffma": N.KNN_EXACT_FFMA}[knn_mode]
    check(lib().nomad_b200_group_index_sharded(group.h, arr, r0.ctypes.data, n_total, C_,
                                               seed & (2**64 - 1), max_iters, tol, workers, k, km,
                                               C.byref(cv), C.byref(gv)))
    m = int(off[n_total])
    return ca, KnnGraph(n_total, k, off, nb[:m], di[:m])


def pca_init_sharded(rows, row0: int, n_total: int, seed: int = 0, fast: bool = False,
                     rank: int = 0, world_size: int = 1, nccl_id: Optional[bytes] = None,
                     ctx: Optional[Context] = None) -> np.ndarray:
    """Row-sharded pca_init (pca.hpp:79-218) for one rank of a multi-process
    run: this rank holds rows [row0, row0 + len(rows)) and gets their layout
    rows; fast=False is bit-identical to pca_init on the whole dataset."""
    dv, keep = _dataset(rows)
    out = np.zeros((dv.rows, 2), np.float64)
    idbuf = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
    check(lib().nomad_b200_pca_init_sharded(_ctx(ctx).h, rank, world_size, idbuf, C.byref(dv),
                                            row0, n_total, seed & (2**64 - 1), int(fast),
                                            out.ctypes.data, N.HOST))
    return out


def group_pca_init_sharded(group: "Group", rows: list, row0: list, n_total: int, seed: int = 0,
                           fast: bool = False) -> list:
    """Row-sharded pca_init over the ranks of a Group (rows[r] on rank r's
    device): the layout rows of every rank's slice, in rank order."""
    views, keeps, outs = [], [], []
    for r in rows:
        v, kp = _dataset(r)
        views.append(v)
        keeps.append(kp)
        outs.append(np.zeros((v.rows, 2), np.float64))
    arr = (N.DatasetView * len(views))(*views)
    r0 = np.ascontiguousarray(row0, np.uint64)
    ptrs = (C.c_void_p * len(outs))(*[o.ctypes.data for o in outs])
    check(lib().nomad_b200_group_pca_init_sharded(group.h, arr, r0.ctypes.data, n_total,
                                                  seed & (2**64 - 1), int(fast), ptrs, N.HOST))
    return outs


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().nomad_b200_nccl_unique_id(buf))
    return buf.raw


def shard_plan(assignment, n_clusters: int, workers: int, world_size: int = 1):
    """shard_clusters (optimizer.hpp:106-144) + the means all-gather slot layout.

    Returns (cluster_to_worker[C], slot_cluster[world, max_slots]) where
    slot_cluster[r, q] is the cluster whose mean rank r sends in slot q
    (0xFFFFFFFF = padding). Host-only; identical to what the trainer uses."""
    a = np.ascontiguousarray(assignment, np.uint32)
    c2w = np.zeros(n_clusters, np.uint32)
    ms = C.c_uint32()
    check(lib().nomad_b200_plan(len(a), n_clusters, a.ctypes.data, workers, world_size,
                                c2w.ctypes.data, None, C.byref(ms)))
    slots = np.zeros(world_size * ms.value, np.uint32)
    check(lib().nomad_b200_plan(len(a), n_clusters, a.ctypes.data, workers, world_size,
                                c2w.ctypes.data, slots.ctypes.data, C.byref(ms)))
    return c2w, slots.reshape(world_size, ms.value)
