// Deterministic replay on the device (K8r): the reference's per-worker draw
// stream (std::mt19937_64 wrapped by Rng, rng.hpp:42-84; optimizer.hpp:
// 254-255, :284-285) generated on the GPU, and the sequential per-worker
// update order (optimizer.hpp:253-304) enforced by dataflow: every draw waits
// only for the latest earlier draw of its worker that touched each of its
// points.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "sgd_kernels.cuh"

namespace nb {

// std::mt19937_64 state: 312 untempered words and the read position (312 =
// the next call twists), the layout of the standard's sequential algorithm.
struct MtState {
  unsigned long long mt[312];
  uint32_t p, pad;
};

// Host mirror (seeding, seek, the rejection fallback). Seeded exactly as
// std::mt19937_64(seed); next() returns the same sequence.
struct Mt64 {
  MtState s;
  void seed(uint64_t v);
  void twist();
  uint64_t next();
  // rng.hpp:49-55 Rng::uniform_index: unbiased bounded draw by rejection
  uint64_t uniform_index(uint64_t n) {
    const uint64_t limit = n * (0xFFFFFFFFFFFFFFFFull / n);
    uint64_t d = next();
    while (d >= limit) d = next();
    return d % n;
  }
};

// Device-side replay schedule of one epoch for the nwl local workers.
struct ReplayDev {
  uint32_t nwl, s, T;          // T = touch slots per draw = 1 + k + s
  const uint32_t* draw_base;   // per worker: first draw index (global over local workers)
  const uint64_t* word_base;   // per worker: first word index
  MtState* st_in;              // per worker: the state at the start of the epoch
  MtState* st_out;             // per worker: the state after the epoch's draws
  unsigned long long* words;   // raw tempered words, worker-major
  uint32_t* heads;             // per draw: local head id
  uint32_t* tails;             // per draw: s local tail ids
  uint32_t* tkey;              // per draw and slot: the slot's local point (n_loc: none /
                               // a repeat within the draw); sorted in place by point
  uint32_t* tval;              // per draw and slot: its flat index i * T + slot
  uint32_t* tkey2;             // radix-sort buffers
  uint32_t* tval2;
  uint32_t* pred;              // per draw and slot: latest earlier draw touching it (none: ~0);
                               // per-thread form only (else nullptr)
  uint2* link;                 // warp form: per draw and slot {latest earlier draw touching
                               // it, the next touch of its point as a flat touch index}
                               // (none: ~0), one 8-byte record (else nullptr)
  double2* mbox;               // per touch: the point's position forwarded by its
                               // predecessor (all-ones bits: not yet); warp form only
  uint32_t n_loc;              // local points (the "none" key)
  uint32_t* reject;            // per worker: a draw hit the rejection branch
  unsigned long long* edges;   // per worker: sum over draws of |N(head)| + s
  uint8_t* done;               // per draw: completed
  uint32_t* ticket;            // dataflow work counter
  uint32_t* stall;             // set if a draw waited beyond the watchdog (never expected)
  const uint32_t* pt_base;     // per local point: draw_base of its worker
  uint32_t total_chunks;       // warps' chunks of draws, worker-interleaved
  uint32_t max_draws, total_draws;
  uint32_t nap_cap;            // longest back-off sleep of a waiting draw (ns)
  uint32_t followers;          // warp form: warps that sum the workers' losses in draw order
                               // while the draws run (0: k_loss_seq afterwards)
  double* wloss;               // per worker: the epoch's loss sum (followers)
};

void launch_mt_words(const ReplayDev& R, const uint64_t* counts, cudaStream_t st);
void launch_replay_map(const ReplayDev& R, const SgdParams& P, const uint32_t* pool,
                       const uint32_t* pool_off, cudaStream_t st);
// touch lists -> stable sort by point (draw order kept inside a point) -> pred
void launch_replay_deps(const ReplayDev& R, const SgdParams& P, void* sort_tmp, size_t sort_bytes,
                        cudaStream_t st);
size_t replay_sort_bytes(uint64_t items, uint32_t n_loc);
void launch_sgd_dataflow(const SgdParams& P, const ReplayDev& R, uint32_t nblocks, size_t smem,
                         cudaStream_t st);
uint32_t dataflow_resident_blocks(size_t smem, int sm_count, uint32_t k, uint32_t s);
// the warp-per-draw form applies when 1 + k + s <= 32; draws claimed per ticket
bool dataflow_warp_form(uint32_t k, uint32_t s);
uint32_t dataflow_draws_per_chunk(uint32_t k, uint32_t s);

}  // namespace nb
