/*
 * nomad_b200.h — C-ABI of the B200-native NOMAD Projection engine
 * (libnomad_b200.so, sm_100a). Plain pointers and sizes only.
 *
 * The reference (/root/reference/proj/include/nomad) is a header-only C++20
 * library of free functions; it has no FFI layer. Each entry point below
 * replaces one reference function (cited as file:line) with the same
 * argument meaning; the C++ shim include/nomad_b200/nomad_b200.hpp re-exposes
 * the reference signatures on top of this ABI, and the Python package
 * paper_2505_15511_b200 binds it with ctypes.
 *
 * Conventions
 *  - Return value: 0 on success, else 1 + ErrorKind in the reference's enum
 *    order (error.hpp:25-36): 1 Io, 2 Dimension, 3 Validation, 4 Schema,
 *    5 Parameter, 6 Config, 7 Degenerate, 8 Divergence, 9 Size, 10 Internal.
 *    CUDA / NCCL failures map to Internal. nomad_b200_last_error() returns the
 *    message (thread-local), e.g. the divergence text of optimizer.hpp:222-225.
 *  - Buffers carry a location flag: NOMAD_B200_HOST (pageable or pinned host
 *    memory) or NOMAD_B200_DEVICE (memory on the context's device, e.g. a
 *    torch CUDA tensor). Device inputs are used in place (no copy).
 *  - Calls are blocking and synchronous w.r.t. the caller (results are ready
 *    on return). A context is not thread-safe; distinct contexts are
 *    independent. No host threads are spawned per epoch.
 *  - There is no CPU fallback: every numeric stage runs in sm_100a kernels.
 */
#ifndef NOMAD_B200_H_
#define NOMAD_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NOMAD_B200_ABI_VERSION 1

enum nomad_b200_status {
  NOMAD_B200_OK = 0,
  NOMAD_B200_ERR_IO = 1,
  NOMAD_B200_ERR_DIMENSION = 2,
  NOMAD_B200_ERR_VALIDATION = 3,
  NOMAD_B200_ERR_SCHEMA = 4,
  NOMAD_B200_ERR_PARAMETER = 5,
  NOMAD_B200_ERR_CONFIG = 6,
  NOMAD_B200_ERR_DEGENERATE = 7,
  NOMAD_B200_ERR_DIVERGENCE = 8,
  NOMAD_B200_ERR_SIZE = 9,
  NOMAD_B200_ERR_INTERNAL = 10
};

enum nomad_b200_location { NOMAD_B200_HOST = 0, NOMAD_B200_DEVICE = 1 };

/* SGD execution mode of the epoch loop (optimizer.hpp:232-307). */
enum nomad_b200_sgd_mode {
  /* Deterministic replay: the reference's per-worker mt19937_64 draw stream
   * (rng.hpp:42-84, optimizer.hpp:254-255, :284-285) generated on the GPU,
   * every draw run once the earlier draws touching its points are done
   * (dataflow); fp64 in the reference's op order, no FMA, non-atomic.
   * Layouts are bit-identical to the reference. */
  NOMAD_B200_SGD_REPLAY = 0,
  /* Throughput mode: counter-based (Philox4x32-10) draws with the reference's
   * distributions, thread-per-head, atomic fp64 scatter-add (Hogwild),
   * bounded heads in flight per shard. Statistically equivalent. */
  NOMAD_B200_SGD_HOGWILD = 1
};

/* kNN distance mode (knn.hpp:65-109). */
enum nomad_b200_knn_mode {
  /* Exact: an fp16 tcgen05 distance filter (top-64 per row) with a rigorous
   * error bound, fp64 j-sequential re-rank and certificate, exhaustive fp64
   * for any uncertified row: ids AND fp64 distances bit-identical to the
   * reference. (k > 56 uses the FFMA filter below.) */
  NOMAD_B200_KNN_EXACT = 0,
  /* bf16 tcgen05 distance contraction (||a||^2+||b||^2-2ab), top-k; report
   * recall@k against the exact mode. Distances returned are fp64 re-ranked. */
  NOMAD_B200_KNN_BF16 = 1,
  /* Exact with the fp32 FFMA direct-difference filter (relative error bound
   * (d+3) u32) instead of the tensor cores; same certificate / fallback. */
  NOMAD_B200_KNN_EXACT_FFMA = 2
};

typedef struct nomad_b200_ctx nomad_b200_ctx;
typedef struct nomad_b200_trainer nomad_b200_trainer;

/* VectorDataset (dataset.hpp:35-44): f32 row-major rows x dims.
 * dtype (appended; 0 from aggregate / zero initialisation = f32):
 * NOMAD_B200_BF16 marks bf16 rows at `data` (the 60M-row configuration's
 * storage). bf16 values widen exactly to f32, so every result equals the f32
 * call on the widened data. Accepted by every entry point that takes a
 * dataset (lsh_init, kmeans_em, build_knn in every mode, knn_recall,
 * pca_init, fit, the metrics). */
#define NOMAD_B200_F32 0
#define NOMAD_B200_BF16 1
typedef struct {
  uint64_t rows;
  uint64_t dims;
  const float* data;
  int32_t location;
  int32_t dtype;
} nomad_b200_dataset_view;

/* ClusterAssignment (kmeans.hpp:32-43). Caller-owned, sized from
 * (rows, n_clusters, dims). centroids may be NULL on output if unwanted. */
typedef struct {
  uint64_t rows;
  uint64_t n_clusters;
  uint64_t dims;
  uint32_t* assignment; /* rows */
  double* centroids;    /* n_clusters * dims */
  uint32_t* sizes;      /* n_clusters */
  int32_t location;
} nomad_b200_clusters;

/* KnnGraph (knn.hpp:31-47), CSR: offsets rows+1; neighbors/distances sized
 * rows*k by the caller (offsets[rows] entries are written). */
typedef struct {
  uint64_t rows;
  uint64_t k;
  uint32_t* offsets;
  uint32_t* neighbors;
  double* distances; /* may be NULL */
  int32_t location;
} nomad_b200_graph;

/* TrainConfig (optimizer.hpp:45-82) plus engine-only fields. */
typedef struct {
  uint64_t epochs;           /* 200 */
  uint64_t k;                /* 15 */
  uint64_t negatives;        /* |M| = 5 */
  uint64_t local_draws;      /* s = 5 */
  uint64_t batch_size;       /* 1024 (a step divisor: step = lr / batch) */
  uint64_t workers;          /* W logical workers (shards) */
  uint64_t n_clusters;       /* 0: auto (optimizer.hpp:73-77) */
  uint64_t seed;
  double lr0;                /* 0: auto n/10 */
  uint64_t kmeans_max_iters; /* 100 */
  double kmeans_tol;         /* < 0: auto (default_kmeans_tol) */
  int32_t approx_all_but_own;/* ApproxMode::AllButOwnCluster */
  int32_t head_only;
  uint64_t checkpoint_every;  /* fit(): layout CSV every N epochs (0: none), optimizer.hpp:463-469 */
  const char* checkpoint_prefix;   /* "<prefix>.epoch<N>.csv" (NULL or "": none) */
  const char* const* checkpoint_ids;    /* row ids (NULL: "0".."n-1", the raw loader's) */
  const char* const* checkpoint_labels; /* label column (NULL: none) */
  /* engine-only */
  int32_t sgd_mode;          /* nomad_b200_sgd_mode */
  int32_t knn_mode;          /* nomad_b200_knn_mode */
  uint32_t hogwild_cap;      /* heads in flight per shard <= shard/cap (0: 16) */
  int32_t hogwild_double_float; /* throughput mode: 0 = f64 position rows, two RED.F64 per
                                row update (default); 1 = double-float rows {hi, lo} (value
                                hi + lo, 48-bit significand), one RED.F32x2 per row update */
  int32_t verbose;           /* per-epoch line to stderr (optimizer.hpp:455-462) */
} nomad_b200_train_config;

/* Fills *cfg with the reference defaults (optimizer.hpp:45-61), replay mode,
 * exact kNN. */
void nomad_b200_default_config(nomad_b200_train_config* cfg);

/* ----------------------------------------------------------- context */
int32_t nomad_b200_create(int32_t device, nomad_b200_ctx** out);
int32_t nomad_b200_destroy(nomad_b200_ctx* ctx);
const char* nomad_b200_last_error(void);
/* Work is issued on this stream (a cudaStream_t); NULL = the context's own. */
int32_t nomad_b200_set_stream(nomad_b200_ctx* ctx, void* cuda_stream);
/* Number of kernels this context has launched so far (evidence counter). */
uint64_t nomad_b200_kernel_launches(const nomad_b200_ctx* ctx);

/* ------------------------------------------- multi-device group (one process)
 * The reference's fit() drives all W workers from one call (one std::thread
 * per worker, optimizer.hpp:327-328, :399-408). A group is the engine's
 * equivalent: one context per entry of `devices`, driven by the calling host
 * thread. Logical workers map to group ranks in contiguous blocks.
 *  - all devices distinct: one NCCL communicator per device (ncclCommInitAll);
 *    the per-epoch means exchange is ncclAllGather over NVLink / NVSwitch.
 *  - all devices equal (e.g. {0,0,0,0}): an in-process loopback exchange
 *    (device copies on one shared stream) — G ranks' trainers on one GPU, for
 *    testing the G-rank math without G GPUs.
 * Mixed lists are rejected (NOMAD_B200_ERR_PARAMETER). */
typedef struct nomad_b200_group nomad_b200_group;
int32_t nomad_b200_group_create(const int32_t* devices, int32_t n_devices,
                                nomad_b200_group** out);
int32_t nomad_b200_group_destroy(nomad_b200_group* g);
/* Ranks in the group, and whether the exchange is the loopback form. */
int32_t nomad_b200_group_size(const nomad_b200_group* g, int32_t* size, int32_t* loopback);
/* Context of rank r (owned by the group; valid until group_destroy). */
int32_t nomad_b200_group_context(nomad_b200_group* g, int32_t rank, nomad_b200_ctx** out);

/* ------------------------------------------------ index build (L2) */
/* kmeans.hpp:157-161 default_kmeans_tol */
int32_t nomad_b200_default_kmeans_tol(nomad_b200_ctx* ctx,
                                      const nomad_b200_dataset_view* data,
                                      double* tol_out);
/* kmeans.hpp:167-250 lsh_init. out->n_clusters = C. */
int32_t nomad_b200_lsh_init(nomad_b200_ctx* ctx,
                            const nomad_b200_dataset_view* data,
                            uint64_t n_clusters, uint64_t seed,
                            nomad_b200_clusters* out);
/* kmeans.hpp:257-296 kmeans_em; inout holds the init and receives the result.
 * qe_trace: NULL or max_iters doubles; iters_out: iterations run (nullable).*/
int32_t nomad_b200_kmeans_em(nomad_b200_ctx* ctx,
                             const nomad_b200_dataset_view* data,
                             nomad_b200_clusters* inout, uint64_t max_iters,
                             double tol, double* qe_trace, uint64_t* iters_out);
/* kmeans_em(data, init, max_iters, default_kmeans_tol(data)) as fit() calls
 * it (optimizer.hpp:337-339). The tolerance is bracketed from a parallel
 * sum and resolved exactly (sequential sum) only if a max_move falls inside
 * the bracket, so the result equals the reference's. */
int32_t nomad_b200_kmeans_em_default_tol(nomad_b200_ctx* ctx,
                                         const nomad_b200_dataset_view* data,
                                         nomad_b200_clusters* inout,
                                         uint64_t max_iters, double* qe_trace,
                                         uint64_t* iters_out);
/* knn.hpp:65-109 build_knn. clusters: assignment + sizes. */
int32_t nomad_b200_build_knn(nomad_b200_ctx* ctx,
                             const nomad_b200_dataset_view* data,
                             const nomad_b200_clusters* clusters, uint64_t k,
                             int32_t knn_mode, nomad_b200_graph* out);

/* Multi-GPU form of build_knn: lists are built only for the rows of the
 * `n_owned` clusters in owned_clusters (host array, e.g. the clusters of this
 * rank's shards from nomad_b200_plan); every other row gets an empty list.
 * Owned rows' lists are identical to build_knn's (clusters are independent,
 * knn.hpp:62-64), and the trainer reads only its own rows. */
int32_t nomad_b200_build_knn_shard(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                   const nomad_b200_clusters* clusters, uint64_t k,
                                   int32_t knn_mode, uint64_t n_owned,
                                   const uint32_t* owned_clusters, nomad_b200_graph* out);
/* recall@k of `graph` against exact lists recomputed (exhaustive fp64) for
 * `sample` rows drawn without replacement from the rows with a non-empty
 * list (0 = all rows). */
int32_t nomad_b200_knn_recall(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                              const nomad_b200_clusters* clusters,
                              const nomad_b200_graph* graph, uint64_t sample, uint64_t seed,
                              double* recall_out);
/* Row-sharded index build (the 60M-row configuration): this
 * rank holds only rows [row0, row0 + rows->rows) of an n_total-row dataset
 * (ranks tile [0, n_total) in rank order). lsh_init + kmeans_em run
 * row-sharded as fit() calls them (optimizer.hpp:336-339; kmeans_tol < 0:
 * default_kmeans_tol): integer counts are all-reduced and every sum the
 * reference accumulates in ascending point id is carried rank to rank, so
 * clusters and centroids are bit-identical to the one-GPU build. Rows then
 * move once to the rank owning their cluster (shard_clusters over `workers`
 * in contiguous rank blocks, optimizer.hpp:106-144) and each rank builds the
 * kNN lists of its clusters (knn.hpp:65-109; identical to the full build's).
 * One process per GPU over NCCL (128-byte nccl_id; NULL when world == 1).
 * Outputs (host, nullable): clusters_out (n_total assignment, centroids,
 * sizes: every rank's copy is the same) and graph_out (CSR over n_total rows
 * holding this rank's lists only; neighbors / distances capacity n_total*k). */
int32_t nomad_b200_index_sharded(nomad_b200_ctx* ctx, int32_t rank, int32_t world,
                                 const void* nccl_id, const nomad_b200_dataset_view* rows,
                                 uint64_t row0, uint64_t n_total, uint64_t n_clusters,
                                 uint64_t seed, uint64_t kmeans_max_iters, double kmeans_tol,
                                 uint64_t workers, uint64_t k, int32_t knn_mode,
                                 nomad_b200_clusters* clusters_out, nomad_b200_graph* graph_out);
/* The same over the ranks of a group (one host thread per rank): rows[r] /
 * row0[r] on rank r's device; graph_out receives every rank's lists. */
int32_t nomad_b200_group_index_sharded(nomad_b200_group* g, const nomad_b200_dataset_view* rows,
                                       const uint64_t* row0, uint64_t n_total,
                                       uint64_t n_clusters, uint64_t seed,
                                       uint64_t kmeans_max_iters, double kmeans_tol,
                                       uint64_t workers, uint64_t k, int32_t knn_mode,
                                       nomad_b200_clusters* clusters_out,
                                       nomad_b200_graph* graph_out);
/* Row-sharded PCA initialisation (pca.hpp:79-218): rank `rank`
 * holds rows [row0, row0 + rows->rows) of an n_total-row dataset and receives
 * those rows' layout (rows->rows x 2, `location`). Every ascending-row sum is
 * carried rank to rank, so fast == 0 is bit-identical to nomad_b200_pca_init
 * on the whole dataset; fast != 0 adds the ranks' covariance sums in rank
 * order (nomad_b200_pca_init_fast's principal plane). NCCL between processes
 * (nccl_id as for nomad_b200_trainer_create; world 1 needs none). */
int32_t nomad_b200_pca_init_sharded(nomad_b200_ctx* ctx, int32_t rank, int32_t world,
                                    const void* nccl_id, const nomad_b200_dataset_view* rows,
                                    uint64_t row0, uint64_t n_total, uint64_t seed, int32_t fast,
                                    double* layout_out, int32_t location);
/* The same over the ranks of a group: rows[r] / row0[r] / layout_out[r] on
 * rank r's device. */
int32_t nomad_b200_group_pca_init_sharded(nomad_b200_group* g, const nomad_b200_dataset_view* rows,
                                          const uint64_t* row0, uint64_t n_total, uint64_t seed,
                                          int32_t fast, double* const* layout_out,
                                          int32_t location);
/* Statistics of the context's last build_knn: rows the tensor-core
 * certificate did not settle, and rows resolved by the exhaustive fp64 pass. */
int32_t nomad_b200_knn_stats(nomad_b200_ctx* ctx, uint64_t* tc_uncertified,
                             uint64_t* exhaustive_rows);
/* Of the tc_uncertified rows, those settled by the sub-cluster stage (exact
 * lists inside sub-clusters + a geometric bound on the other sub-clusters). */
int32_t nomad_b200_knn_subcluster_rows(nomad_b200_ctx* ctx, uint64_t* rows);

/* ------------------------------------------- final-map quality metrics */
/* metrics.hpp:113-168 neighborhood_preservation on the GPU. Same evaluated
 * points (sample == 0 or >= rows: all; else partial Fisher-Yates on the
 * reference stream stream_seed(seed, "np")), exact high-d neighbours by
 * (reference fp64 distance, id), exact 2-D neighbours, overlaps accumulated
 * in evaluation order: value and std_error are bit-identical to the
 * reference's. layout: rows x 2 f64 at layout_location. 1 <= k <= 1024,
 * k < rows (else NOMAD_B200_ERR_PARAMETER); k > 56 searches the high-d rows
 * exhaustively in fp64. std_error may be NULL. */
int32_t nomad_b200_neighborhood_preservation(nomad_b200_ctx* ctx,
                                             const nomad_b200_dataset_view* high,
                                             const double* layout, int32_t layout_location,
                                             uint64_t k, uint64_t sample, uint64_t seed,
                                             double* value, double* std_error);
/* metrics.hpp:174-200 neighborhood_preservation_ann on the GPU: high-d
 * neighbourhoods from a prebuilt within-cluster graph (first min(k, |list|)
 * ids), exact 2-D neighbours of every row on the device; bit-identical value.
 * 1 <= k <= 1024, k < rows. */
int32_t nomad_b200_neighborhood_preservation_ann(nomad_b200_ctx* ctx,
                                                 const nomad_b200_graph* graph,
                                                 const double* layout, int32_t layout_location,
                                                 uint64_t k, double* value);
/* metrics.hpp:205-243 random_triplet_accuracy on the GPU: triplets drawn on
 * the host from the reference stream stream_seed(seed, "tri"), distances and
 * the agreement count on the device; bit-identical value / std_error. */
int32_t nomad_b200_random_triplet_accuracy(nomad_b200_ctx* ctx,
                                           const nomad_b200_dataset_view* high,
                                           const double* layout, int32_t layout_location,
                                           uint64_t n_triplets, uint64_t seed, double* value,
                                           double* std_error);

/* --------------------------------------------- epoch loop (L3 + L4) */
/* The setup half of fit() (optimizer.hpp:342-386): build_affinity,
 * shard_clusters, make_noise_model, worker states, means of the init layout.
 * graph: CSR; clusters: assignment + n_clusters (sizes recomputed).
 * init_layout: rows x 2 f64 (e.g. pca_init). Multi-GPU: rank/world_size and
 * a 128-byte ncclUniqueId (nccl_id may be NULL when world_size == 1). Every
 * rank passes the full index; rank r trains workers
 * [r*W/world, (r+1)*W/world) (W % world_size == 0). */
int32_t nomad_b200_trainer_create(nomad_b200_ctx* ctx,
                                  const nomad_b200_graph* graph,
                                  const nomad_b200_clusters* clusters,
                                  const double* init_layout,
                                  int32_t init_location,
                                  const nomad_b200_train_config* cfg,
                                  int32_t rank, int32_t world_size,
                                  const void* nccl_id,
                                  nomad_b200_trainer** out);
/* The same trainer over a group: rank r of the group trains workers
 * [r*W/G, (r+1)*W/G) on the group's r-th context, and every trainer_* call
 * below drives all G ranks (one epoch = every rank's SGD, then one means
 * exchange). Results are those of a G-process run: replay mode is
 * bit-identical for every G at fixed W. Inputs may be host buffers or
 * device buffers on rank 0's device. */
int32_t nomad_b200_group_trainer_create(nomad_b200_group* g,
                                        const nomad_b200_graph* graph,
                                        const nomad_b200_clusters* clusters,
                                        const double* init_layout,
                                        int32_t init_location,
                                        const nomad_b200_train_config* cfg,
                                        nomad_b200_trainer** out);
int32_t nomad_b200_trainer_destroy(nomad_b200_trainer* tr);
/* Ranks driven by this trainer object (1 for trainer_create, G for a group). */
int32_t nomad_b200_trainer_ranks(nomad_b200_trainer* tr, int32_t* ranks);
/* Runs the next n_epochs epochs of the cfg->epochs schedule
 * (optimizer.hpp:388-470): SGD epoch, means all-gather, mean loss.
 * epoch_loss: NULL or n_epochs doubles. */
int32_t nomad_b200_trainer_run(nomad_b200_trainer* tr, uint64_t n_epochs,
                               double* epoch_loss);
/* Current layout in ORIGINAL point order (rows x 2 f64). On a multi-GPU
 * trainer only this rank's points are written (others untouched). */
int32_t nomad_b200_trainer_layout(nomad_b200_trainer* tr, double* out,
                                  int32_t location);
/* Current all-gathered ClusterMeans snapshot (objective.hpp:65-73):
 * means n_clusters x 2, counts n_clusters; either may be NULL. */
int32_t nomad_b200_trainer_means(nomad_b200_trainer* tr, double* means,
                                 uint32_t* counts);
/* CommLog counters (optimizer.hpp:178-189): totals since creation. */
int32_t nomad_b200_trainer_comm(nomad_b200_trainer* tr, uint64_t* epochs,
                                uint64_t* messages, uint64_t* payload_doubles,
                                uint64_t* payload_counts);
/* Replace the positions (rows x 2, ORIGINAL order) and re-gather the means
 * snapshot (the layout handed to the epoch loop, optimizer.hpp:353/:384). */
int32_t nomad_b200_trainer_set_layout(nomad_b200_trainer* tr, const double* layout,
                                      int32_t location);
/* Device time (CUDA events on the launching stream) accumulated over every
 * epoch run so far: the SGD kernel, and the means + all-gather step. */
int32_t nomad_b200_trainer_timing(nomad_b200_trainer* tr, double* sgd_ms,
                                  double* means_ms, uint64_t* epochs);
/* Continue the epoch schedule at `epoch` (resume: trainer_set_layout with a
 * checkpoint written after `epoch` epochs, then seek). Throughput mode: any
 * epoch (Philox draws are keyed by epoch); replay mode: forward only, the
 * workers' mt19937_64 streams are advanced past the skipped draws, so the
 * resumed run is bit-identical to an uninterrupted one. */
int32_t nomad_b200_trainer_seek(nomad_b200_trainer* tr, uint64_t epoch);
/* Epochs completed and edge-updates applied (sum over heads of |N(h)|+s). */
int32_t nomad_b200_trainer_progress(nomad_b200_trainer* tr,
                                    uint64_t* epochs_done,
                                    uint64_t* edge_updates);

/* pca.hpp:79-218 pca_init on the GPU, bit-identical to the reference: every
 * covariance apply is X_c^T (X_c v) / n in the reference's summation orders;
 * the vector algebra, Rng stream, sign rule and rank-1 jitter are the
 * reference's. layout_out: rows x 2 f64. */
int32_t nomad_b200_pca_init(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                            uint64_t seed, double* layout_out, int32_t location);
/* The same algorithm with the covariance sums formed once (one fp64 pass
 * over the centred data) and each apply a d x d product: the basis agrees
 * with the reference's to rounding, so the layout spans the same principal
 * plane, but its in-plane orientation may differ (pca.hpp:150-165 rotates by
 * an angle computed from rounding-level quantities). ~1 pass over the data
 * instead of ~2 per power iteration (1M x 768: 0.3-0.8 s vs 41 s). fit()
 * uses it in throughput (hogwild) mode. */
int32_t nomad_b200_pca_init_fast(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                 uint64_t seed, double* layout_out, int32_t location);

/* --------------------------------------------------- fit (L4) */
/* optimizer.hpp:327-482 fit. init_layout: the PCA initialisation
 * (pca.hpp:79, rows x 2; NULL = computed on the GPU by power iteration).
 * layout_out: rows x 2 f64. Report pointers may be NULL. */
int32_t nomad_b200_fit(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                       const nomad_b200_train_config* cfg,
                       const double* init_layout, double* layout_out,
                       nomad_b200_clusters* clusters_out,
                       nomad_b200_graph* graph_out, double* epoch_loss_out);

/* Everything fit() produced besides the layout (FitReport,
 * optimizer.hpp:312-321), each taken from the engine's own outputs. Every
 * pointer may be NULL; host buffers unless the view says otherwise. */
typedef struct {
  nomad_b200_clusters* clusters;  /* ClusterAssignment (kmeans.hpp:32-43) */
  nomad_b200_graph* graph;        /* KnnGraph (knn.hpp:31-47) */
  double* epoch_mean_loss;        /* epochs */
  double* pca;                    /* rows x 2: the init layout the epochs started from */
  double* final_means;            /* n_clusters x 2: the last all-gathered ClusterMeans */
  uint32_t* cluster_to_worker;    /* n_clusters: ShardPlan (optimizer.hpp:94-144) */
  double* affinity_weights;       /* rows * k: p(j|i) per edge, CSR as the graph (affinity.hpp:65-84) */
  uint32_t* eligible_heads;       /* rows: points with >= 1 neighbour, ascending */
  /* out */
  uint64_t n_clusters;            /* resolved C (optimizer.hpp:73-77) */
  uint64_t n_eligible;
  uint64_t comm_epochs, comm_messages, comm_payload_doubles, comm_payload_counts; /* CommLog */
} nomad_b200_fit_report;

/* fit() with the whole report, on one context (group == NULL) or on a group
 * (ctx == NULL: the index is built on rank 0's device, the epochs run on
 * every rank of the group). init_layout NULL: the GPU PCA (bit-identical in
 * replay mode, the precomputed-covariance form in throughput mode). */
int32_t nomad_b200_fit_ex(nomad_b200_ctx* ctx, nomad_b200_group* group,
                          const nomad_b200_dataset_view* data,
                          const nomad_b200_train_config* cfg, const double* init_layout,
                          double* layout_out, nomad_b200_fit_report* report);

/* ----------------------------------------------------------- data I/O */
/* dataset.hpp:122-173 load_vectors_raw: little-endian f32 row-major file;
 * rows or dims may be 0 (derived from the file size; both given = strict).
 * Same checks and messages (Io / Parameter / Dimension / Validation: first
 * non-finite value in row-major order). out == NULL: shape query only.
 * out_location DEVICE streams the file through pinned buffers into device
 * memory (ctx required; the finiteness scan runs on the GPU). */
int32_t nomad_b200_load_vectors_raw(nomad_b200_ctx* ctx, const char* path, uint64_t rows,
                                    uint64_t dims, float* out, int32_t out_location,
                                    uint64_t* rows_out, uint64_t* dims_out);
/* dataset.hpp:223-250 save_layout: `id,x,y[,label]`, %.17g, byte-identical
 * to the reference (formatted on all host cores). layout: host rows x 2.
 * ids NULL: "0".."rows-1"; labels NULL: no label column. */
int32_t nomad_b200_save_layout_csv(const char* path, const double* layout, uint64_t rows,
                                   const char* const* ids, const char* const* labels);
/* Raw little-endian f64 rows x 2 (16 bytes per row, no header). */
int32_t nomad_b200_save_layout_f64(const char* path, const double* layout, uint64_t rows);

/* ------------------------------------------- helpers (multi-GPU, data) */
/* Host-only: shard_clusters' LPT plan (optimizer.hpp:106-144) for `workers`
 * logical workers mapped to `world` ranks in contiguous blocks, and the slot
 * layout of the per-epoch means all-gather: slot_cluster[world * max_slots]
 * holds the cluster id of each rank's slot (UINT32_MAX = padding; NULL to
 * skip). cluster_to_worker: n_clusters entries. */
int32_t nomad_b200_plan(uint64_t n, uint64_t n_clusters, const uint32_t* assignment,
                        uint64_t workers, int32_t world, uint32_t* cluster_to_worker,
                        uint32_t* slot_cluster, uint32_t* max_slots);
/* ncclGetUniqueId into 128 bytes (rank 0 calls it, then broadcasts). */
int32_t nomad_b200_nccl_unique_id(void* out128);
/* Synthetic Gaussian mixture on the device: centres
 * ~N(0, spread^2), x_i = c_{i mod blobs} + N(0,1), Philox4x32-10 streams.
 * out: rows*dims f32 on the device. */
int32_t nomad_b200_generate_mixture(nomad_b200_ctx* ctx, uint64_t rows,
                                    uint64_t dims, uint64_t blobs,
                                    double spread, uint64_t seed, float* out);
/* The same mixture as bf16 rows (each f32 value rounded to nearest even):
 * the storage of the 60M x 768 bf16 configuration. out: rows*dims bf16. */
int32_t nomad_b200_generate_mixture_bf16(nomad_b200_ctx* ctx, uint64_t rows,
                                         uint64_t dims, uint64_t blobs,
                                         double spread, uint64_t seed, void* out);

/* Rows [row0, row0 + rows) of the same mixture (one rank's share of a
 * row-sharded dataset; identical to those rows of the full matrix). dtype:
 * NOMAD_B200_F32 or NOMAD_B200_BF16. */
int32_t nomad_b200_generate_mixture_rows(nomad_b200_ctx* ctx, uint64_t row0, uint64_t rows,
                                         uint64_t dims, uint64_t blobs, double spread,
                                         uint64_t seed, int32_t dtype, void* out);

/* Diagnostic: one 128 x 128 bf16 tile product D = A B^T through the same
 * TMA + tcgen05.mma + TMEM path the bf16 kNN uses (rows rounded to bf16). */
/* Debug / unit path of the fast PCA: S = sum_i (x_i - mean)(x_i - mean)^T
 * (out_host: d x d). */
int32_t nomad_b200_debug_cov(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                             const double* mean_host, double* out_host);
int32_t nomad_b200_debug_tc_gemm(nomad_b200_ctx* ctx, const float* host_rows, uint64_t rows,
                                 uint64_t d, uint32_t a0, uint32_t b0, float* out128x128);

#ifdef __cplusplus
}
#endif
#endif /* NOMAD_B200_H_ */
