"""ctypes binding of libnomad_b200.so (include/nomad_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()``
(paper_2505_15511_b200/csrc/Makefile). There is no fallback: if the library is
missing or cannot load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NOMAD_B200_LIB") or os.path.join(HERE, "libnomad_b200.so")

KINDS = ["Io", "Dimension", "Validation", "Schema", "Parameter", "Config",
         "Degenerate", "Divergence", "Size", "Internal"]

HOST, DEVICE = 0, 1
SGD_REPLAY, SGD_HOGWILD = 0, 1
KNN_EXACT, KNN_BF16, KNN_EXACT_FFMA = 0, 1, 2


class NomadError(RuntimeError):
    """nomad::Error (error.hpp:38-47): carries the ErrorKind name."""

    def __init__(self, kind: str, message: str):
        super().__init__(message)
        self.kind = kind
        self.message = message


F32, BF16 = 0, 1  # nomad_b200_dataset_view.dtype


class DatasetView(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("dims", C.c_uint64), ("data", C.c_void_p),
                ("location", C.c_int32), ("dtype", C.c_int32)]


class ClustersView(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("n_clusters", C.c_uint64), ("dims", C.c_uint64),
                ("assignment", C.c_void_p), ("centroids", C.c_void_p), ("sizes", C.c_void_p),
                ("location", C.c_int32)]


class GraphView(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("k", C.c_uint64), ("offsets", C.c_void_p),
                ("neighbors", C.c_void_p), ("distances", C.c_void_p), ("location", C.c_int32)]


class TrainConfigC(C.Structure):
    _fields_ = [("epochs", C.c_uint64), ("k", C.c_uint64), ("negatives", C.c_uint64),
                ("local_draws", C.c_uint64), ("batch_size", C.c_uint64),
                ("workers", C.c_uint64), ("n_clusters", C.c_uint64), ("seed", C.c_uint64),
                ("lr0", C.c_double), ("kmeans_max_iters", C.c_uint64),
                ("kmeans_tol", C.c_double), ("approx_all_but_own", C.c_int32),
                ("head_only", C.c_int32), ("checkpoint_every", C.c_uint64),
                ("checkpoint_prefix", C.c_char_p), ("checkpoint_ids", C.c_void_p),
                ("checkpoint_labels", C.c_void_p), ("sgd_mode", C.c_int32), ("knn_mode", C.c_int32),
                ("hogwild_cap", C.c_uint32), ("hogwild_double_float", C.c_int32),
                ("verbose", C.c_int32)]


class FitReportC(C.Structure):
    _fields_ = [("clusters", C.c_void_p), ("graph", C.c_void_p), ("epoch_mean_loss", C.c_void_p),
                ("pca", C.c_void_p), ("final_means", C.c_void_p),
                ("cluster_to_worker", C.c_void_p), ("affinity_weights", C.c_void_p),
                ("eligible_heads", C.c_void_p), ("n_clusters", C.c_uint64),
                ("n_eligible", C.c_uint64), ("comm_epochs", C.c_uint64),
                ("comm_messages", C.c_uint64), ("comm_payload_doubles", C.c_uint64),
                ("comm_payload_counts", C.c_uint64)]


_vp = C.c_void_p
_SIGS = {
    "nomad_b200_last_error": (C.c_char_p, []),
    "nomad_b200_default_config": (None, [C.POINTER(TrainConfigC)]),
    "nomad_b200_create": (C.c_int32, [C.c_int32, C.POINTER(_vp)]),
    "nomad_b200_destroy": (C.c_int32, [_vp]),
    "nomad_b200_set_stream": (C.c_int32, [_vp, _vp]),
    "nomad_b200_kernel_launches": (C.c_uint64, [_vp]),
    "nomad_b200_default_kmeans_tol": (C.c_int32, [_vp, C.POINTER(DatasetView),
                                                  C.POINTER(C.c_double)]),
    "nomad_b200_lsh_init": (C.c_int32, [_vp, C.POINTER(DatasetView), C.c_uint64, C.c_uint64,
                                        C.POINTER(ClustersView)]),
    "nomad_b200_kmeans_em": (C.c_int32, [_vp, C.POINTER(DatasetView), C.POINTER(ClustersView),
                                         C.c_uint64, C.c_double, _vp,
                                         C.POINTER(C.c_uint64)]),
    "nomad_b200_kmeans_em_default_tol": (C.c_int32, [_vp, C.POINTER(DatasetView),
                                                     C.POINTER(ClustersView), C.c_uint64, _vp,
                                                     C.POINTER(C.c_uint64)]),
    "nomad_b200_build_knn": (C.c_int32, [_vp, C.POINTER(DatasetView), C.POINTER(ClustersView),
                                         C.c_uint64, C.c_int32, C.POINTER(GraphView)]),
    "nomad_b200_knn_recall": (C.c_int32, [_vp, C.POINTER(DatasetView), C.POINTER(ClustersView),
                                          C.POINTER(GraphView), C.c_uint64, C.c_uint64,
                                          C.POINTER(C.c_double)]),
    "nomad_b200_knn_stats": (C.c_int32, [_vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "nomad_b200_knn_subcluster_rows": (C.c_int32, [_vp, C.POINTER(C.c_uint64)]),
    "nomad_b200_neighborhood_preservation": (C.c_int32, [_vp, C.POINTER(DatasetView), _vp, C.c_int32,
                                                         C.c_uint64, C.c_uint64, C.c_uint64,
                                                         C.POINTER(C.c_double),
                                                         C.POINTER(C.c_double)]),
    "nomad_b200_neighborhood_preservation_ann": (C.c_int32, [_vp, C.POINTER(GraphView), _vp,
                                                             C.c_int32, C.c_uint64,
                                                             C.POINTER(C.c_double)]),
    "nomad_b200_random_triplet_accuracy": (C.c_int32, [_vp, C.POINTER(DatasetView), _vp, C.c_int32,
                                                       C.c_uint64, C.c_uint64,
                                                       C.POINTER(C.c_double),
                                                       C.POINTER(C.c_double)]),
    "nomad_b200_trainer_create": (C.c_int32, [_vp, C.POINTER(GraphView), C.POINTER(ClustersView),
                                              _vp, C.c_int32, C.POINTER(TrainConfigC),
                                              C.c_int32, C.c_int32, _vp, C.POINTER(_vp)]),
    "nomad_b200_trainer_destroy": (C.c_int32, [_vp]),
    "nomad_b200_group_create": (C.c_int32, [_vp, C.c_int32, C.POINTER(_vp)]),
    "nomad_b200_group_destroy": (C.c_int32, [_vp]),
    "nomad_b200_group_size": (C.c_int32, [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "nomad_b200_group_context": (C.c_int32, [_vp, C.c_int32, C.POINTER(_vp)]),
    "nomad_b200_group_trainer_create": (C.c_int32, [_vp, C.POINTER(GraphView),
                                                    C.POINTER(ClustersView), _vp, C.c_int32,
                                                    C.POINTER(TrainConfigC), C.POINTER(_vp)]),
    "nomad_b200_trainer_ranks": (C.c_int32, [_vp, C.POINTER(C.c_int32)]),
    "nomad_b200_trainer_run": (C.c_int32, [_vp, C.c_uint64, _vp]),
    "nomad_b200_trainer_layout": (C.c_int32, [_vp, _vp, C.c_int32]),
    "nomad_b200_trainer_means": (C.c_int32, [_vp, _vp, _vp]),
    "nomad_b200_trainer_comm": (C.c_int32, [_vp] + [C.POINTER(C.c_uint64)] * 4),
    "nomad_b200_trainer_set_layout": (C.c_int32, [_vp, _vp, C.c_int32]),
    "nomad_b200_trainer_timing": (C.c_int32, [_vp, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                              C.POINTER(C.c_uint64)]),
    "nomad_b200_trainer_progress": (C.c_int32, [_vp] + [C.POINTER(C.c_uint64)] * 2),
    "nomad_b200_pca_init": (C.c_int32, [_vp, C.POINTER(DatasetView), C.c_uint64, _vp, C.c_int32]),
    "nomad_b200_fit": (C.c_int32, [_vp, C.POINTER(DatasetView), C.POINTER(TrainConfigC), _vp,
                                   _vp, C.POINTER(ClustersView), C.POINTER(GraphView), _vp]),
    "nomad_b200_fit_ex": (C.c_int32, [_vp, _vp, C.POINTER(DatasetView), C.POINTER(TrainConfigC),
                                      _vp, _vp, C.POINTER(FitReportC)]),
    "nomad_b200_index_sharded": (C.c_int32, [_vp, C.c_int32, C.c_int32, _vp, C.POINTER(DatasetView),
                                             C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                             C.c_uint64, C.c_double, C.c_uint64, C.c_uint64,
                                             C.c_int32, C.POINTER(ClustersView),
                                             C.POINTER(GraphView)]),
    "nomad_b200_group_index_sharded": (C.c_int32, [_vp, C.POINTER(DatasetView), _vp, C.c_uint64,
                                                   C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                                   C.c_uint64, C.c_uint64, C.c_int32,
                                                   C.POINTER(ClustersView), C.POINTER(GraphView)]),
    "nomad_b200_pca_init_sharded": (C.c_int32, [_vp, C.c_int32, C.c_int32, _vp,
                                                C.POINTER(DatasetView), C.c_uint64, C.c_uint64,
                                                C.c_uint64, C.c_int32, _vp, C.c_int32]),
    "nomad_b200_group_pca_init_sharded": (C.c_int32, [_vp, C.POINTER(DatasetView), _vp,
                                                      C.c_uint64, C.c_uint64, C.c_int32, _vp,
                                                      C.c_int32]),
    "nomad_b200_generate_mixture_rows": (C.c_int32, [_vp, C.c_uint64, C.c_uint64, C.c_uint64,
                                                     C.c_uint64, C.c_double, C.c_uint64, C.c_int32,
                                                     _vp]),
    "nomad_b200_plan": (C.c_int32, [C.c_uint64, C.c_uint64, _vp, C.c_uint64, C.c_int32, _vp, _vp,
                                    C.POINTER(C.c_uint32)]),
    "nomad_b200_debug_tc_gemm": (C.c_int32, [_vp, _vp, C.c_uint64, C.c_uint64, C.c_uint32,
                                             C.c_uint32, _vp]),
    "nomad_b200_nccl_unique_id": (C.c_int32, [_vp]),
    "nomad_b200_trainer_seek": (C.c_int32, [_vp, C.c_uint64]),
    "nomad_b200_debug_cov": (C.c_int32, [_vp, C.POINTER(DatasetView), _vp, _vp]),
    "nomad_b200_pca_init_fast": (C.c_int32, [_vp, C.POINTER(DatasetView), C.c_uint64, _vp,
                                             C.c_int32]),
    "nomad_b200_build_knn_shard": (C.c_int32, [_vp, C.POINTER(DatasetView), C.POINTER(ClustersView),
                                               C.c_uint64, C.c_int32, C.c_uint64, _vp,
                                               C.POINTER(GraphView)]),
    "nomad_b200_load_vectors_raw": (C.c_int32, [_vp, C.c_char_p, C.c_uint64, C.c_uint64, _vp,
                                                C.c_int32, C.POINTER(C.c_uint64),
                                                C.POINTER(C.c_uint64)]),
    "nomad_b200_save_layout_csv": (C.c_int32, [C.c_char_p, _vp, C.c_uint64, _vp, _vp]),
    "nomad_b200_save_layout_f64": (C.c_int32, [C.c_char_p, _vp, C.c_uint64]),
    "nomad_b200_generate_mixture": (C.c_int32, [_vp, C.c_uint64, C.c_uint64, C.c_uint64,
                                                C.c_double, C.c_uint64, _vp]),
    "nomad_b200_generate_mixture_bf16": (C.c_int32, [_vp, C.c_uint64, C.c_uint64, C.c_uint64,
                                                C.c_double, C.c_uint64, _vp]),
}

EXPORTED = tuple(_SIGS)
_lib = None


def build(force: bool = False) -> str:
    """Compile libnomad_b200.so in-tree (nvcc, sm_100a)."""
    if force or not os.path.exists(LIB_PATH):
        out = subprocess.run(["make", "-C", os.path.join(HERE, "csrc"), "-j8"],
                             capture_output=True, text=True)
        if out.returncode != 0:
            raise RuntimeError("libnomad_b200 build failed:\n" + out.stdout[-4000:] +
                               out.stderr[-4000:])
    return LIB_PATH


def lib() -> C.CDLL:
    """The loaded library; raises if it is not built (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().nomad_b200_last_error().decode()
        raise NomadError(KINDS[rc - 1] if 1 <= rc <= len(KINDS) else "Internal", msg)
