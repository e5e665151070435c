// Device side of the epoch loop: the SGD kernels (K8r replay, K8p hogwild) and
// the cluster-means kernels (K9). Reference: optimizer.hpp:215-307 (worker
// epoch, apply_update), objective.hpp:36-41/113-145/178-237 (Cauchy kernel,
// noise terms, analytic gradient), optimizer.hpp:411-442 (means all-gather).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "philox.cuh"

namespace nb {

// Per logical worker (shard) on this rank. Points of worker w are the
// contiguous local ids [pstart, pstart + npts), grouped by cluster (ascending
// cluster id), ascending original id inside each cluster.
struct WorkerDev {
  uint32_t pstart, npts;      // local point range
  uint32_t elig_off, n_elig;  // eligible heads (local ids) in elig[]
  uint32_t rem_off, n_rem;    // remote cells R~ (RemoteClusters mode)
  uint32_t draws;             // heads drawn this epoch (= n_elig)
  uint32_t chunk0;            // unused (kept for layout)
  uint32_t all_elig;          // eligible == all points (head = pstart + idx)
  uint32_t id;                // global worker id
  double local_mass;          // optimizer.hpp:369-370
};

// A cluster owned by this rank: local ids [start, start + count).
struct LocalCluster {
  uint32_t start, count, gid, worker;  // worker = local worker index
};

struct SgdParams {
  double2* pos;                 // local positions (f64 x, y; hogwild: double-float rows)
  const uint32_t* ell;          // local ids, kpad per row
  const uint8_t* ncnt;          // neighbour count per row (nullptr: all == k)
  const double* wtab;           // (k+1) x k inverse-rank weights, row = count
  const uint32_t* elig;         // eligible heads, local ids, worker-major
  const WorkerDev* workers;
  const double2* means;         // all C cluster means (stale snapshot)
  const uint32_t* remote_ids;   // concat per worker (global cluster ids)
  const double* remote_probs;   // p(m in r), parallel
  const uint32_t* cl_of;        // local cluster index per local point (AllButOwn)
  const LocalCluster* lclusters;
  const double* cell_probs;     // global C: size_r / n
  double* loss_acc;             // per local worker
  unsigned long long* edge_acc; // per local worker: sum of |N(h)| + s
  unsigned long long* diverge;  // first offending key (hogwild: one; replay: one per local
                                // worker, (t * stride + u) << 32 | local point)
  uint32_t n_workers, kpad, k, s, m_total, n_clusters;
  int head_only, all_but_own;
  int double_float;             // hogwild: 1 = double-float rows (1 RED.F32x2), 0 = f64 rows (2 RED.F64)
  uint32_t max_cells;           // hogwild: capacity of the shared cell table (per worker row of the global tables)
  // cell tables in global memory when they do not fit in shared memory
  // (many clusters, e.g. the reference's auto C = ceil(n / 4096) at 60M rows)
  int gcells;                   // 1: hogwild reads gcell_mu / gcell_w, replay reads cm3
  const double2* gcell_mu;      // hogwild: [local worker][max_cells] cell means
  const double* gcell_w;        // hogwild: [local worker][max_cells] weights M p_r
  const double* cm3;            // replay: [C][3] = mu.x, mu.y, p_r
  double step;
  uint64_t epoch;
  uint32_t seed_lo, seed_hi;
  // hogwild dynamic schedule (chunks of chunk_heads draws, worker-major)
  uint32_t* chunk_counter;
  uint32_t total_chunks, chunk_heads;
  const uint2* chunk_map;       // chunk -> (local worker, chunk within the worker)
  // replay (replay.cu)
  double* loss_slot;            // per worker-draw loss, indexed by worker base + t
  const uint32_t* wk_draw_base; // per worker: base into loss_slot
};

// Host launchers (sgd.cu).
void launch_loss_seq(const double* slot, const uint32_t* base, const WorkerDev* wk, uint32_t nw,
                     double* out, cudaStream_t st);
void launch_sgd_hogwild(const SgdParams& P, uint32_t nblocks, size_t smem, cudaStream_t st);
uint32_t hogwild_resident_blocks(uint32_t kpad, uint32_t s, size_t smem, int sm_count);
uint32_t hogwild_group_size(uint32_t kpad, uint32_t s);
uint32_t hogwild_chunk_rounds();
void launch_means_exact(const double2* pos, const LocalCluster* lc, uint32_t ncl, double* slot,
                        cudaStream_t st);
void launch_means_chunk(double2* pos, bool df, const LocalCluster* lc, uint32_t ncl, uint32_t chunk,
                        const uint32_t* chunk_off, uint32_t nchunks, double* sums,
                        unsigned long long* diverge, unsigned long long tag, cudaStream_t st);
// f64 rows <-> double-float rows {hi.x, hi.y, lo.x, lo.y}, in place.
void launch_pos_df(double2* pos, uint32_t n, bool to_df, cudaStream_t st);
void launch_means_finalize(double* sums, const LocalCluster* lc, uint32_t ncl, double* slot,
                           cudaStream_t st);
void launch_means_unpack(const double* recv, const uint32_t* slot_gid, uint32_t nslots,
                         double2* means, cudaStream_t st);
// bad: first local row whose list is longer than k or names a point outside
// the row's own worker shard (optimizer.hpp:292-300 ownership asserts).
void launch_build_ell(const uint32_t* offsets, const uint32_t* nbrs, const uint32_t* orig_of,
                      const uint32_t* new_of, const uint32_t* cl_of, const LocalCluster* lcl,
                      uint32_t n_loc, uint32_t k, uint32_t kpad, uint32_t* ell, uint8_t* ncnt,
                      unsigned long long* bad, cudaStream_t st);
// Per-epoch cell tables for the global-memory form (gcells): per local worker
// its remote cells (or all cells, AllButOwn) as mean + weight M p_r, and the
// [C][3] table of the replay kernel.
void launch_cell_tables(const double2* means, const WorkerDev* wk, uint32_t nwl,
                        const uint32_t* remote_ids, const double* remote_probs,
                        const double* cell_probs, uint32_t C, int all_but_own, double M,
                        uint32_t stride, double2* gmu, double* gw, double* cm3, cudaStream_t st);
void launch_scatter_layout(const double2* pos, const uint32_t* orig_of, uint32_t n_loc,
                           double2* out, cudaStream_t st);
void launch_gather_layout(const double2* in, const uint32_t* orig_of, uint32_t n_loc,
                          double2* pos, cudaStream_t st);

}  // namespace nb
