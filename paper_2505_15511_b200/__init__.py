"""B200-native NOMAD Projection engine (arxiv 2505.15511 hot path).

Drop-in for the reference library's index build + epoch loop
(/root/reference/proj/include/nomad): hand-written sm_100a kernels behind the
C-ABI in include/nomad_b200.h (libnomad_b200.so), bound here with ctypes.
"""
from ._native import NomadError, build, lib, EXPORTED  # noqa: F401
from .api import (ClusterAssignment, CommLog, ConditionalAffinity, Context, FitReport,  # noqa: F401
                  Group, KnnGraph, ShardPlan,
                  TrainConfig, Trainer, build_knn, default_kmeans_tol, fit,
                  kmeans_em_default_tol, knn_recall, pca_init, shard_plan,
                  generate_mixture, generate_mixture_rows, group_index_sharded,
                  group_pca_init_sharded, pca_init_sharded,
                  index_sharded, kmeans_em, lsh_init, nccl_unique_id,
                  neighborhood_preservation, neighborhood_preservation_ann,
                  random_triplet_accuracy,
                  load_vectors_raw, save_layout, save_layout_f64)
