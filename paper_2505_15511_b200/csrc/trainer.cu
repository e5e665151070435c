// Host orchestration of the epoch loop: the setup half of fit()
// (optimizer.hpp:342-386), the epoch loop (:388-470) and the cross-shard
// means all-gather (:411-442) over NCCL. All numerics run in sgd.cu kernels;
// the host builds the shard plan / local numbering (O(n) integer work), and,
// in replay mode only, expands the reference's mt19937_64 draw stream into a
// level-ordered tape (the RNG itself is the reference's integer stream).
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <type_traits>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numeric>
#include <random>

#include "common.cuh"
#include "plan.cuh"
#include "sgd_kernels.cuh"

using namespace nb;

namespace {

#define NB_NCCL(call)                                                          \
  do {                                                                         \
    ncclResult_t r_ = (call);                                                  \
    if (r_ != ncclSuccess)                                                     \
      ::nb::fail(::nb::kInternal, std::string("NCCL error: ") + ncclGetErrorString(r_)); \
  } while (0)

// rng.hpp:25-34
uint64_t mix_seed(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
uint64_t stream_seed(uint64_t base, uint64_t stream) { return mix_seed(base ^ mix_seed(stream)); }

// rng.hpp:49-55 — the reference's unbiased bounded draw on mt19937_64.
inline uint64_t uniform_index(std::mt19937_64& g, uint64_t n) {
  const uint64_t limit = n * (0xFFFFFFFFFFFFFFFFull / n);
  uint64_t d = g();
  while (d >= limit) d = g();
  return d % n;
}

// affinity.hpp:32-42 inverse-rank weights (host libm exp, as the reference).
std::vector<double> inverse_rank_weights(uint64_t k) {
  std::vector<double> w(k);
  double total = 0.0;
  for (uint64_t t = 1; t <= k; ++t) {
    w[t - 1] = std::exp(1.0 / static_cast<double>(t));
    total += w[t - 1];
  }
  for (double& x : w) x /= total;
  return w;
}

template <class T>
void upload(DBuf<T>& d, const std::vector<T>& h, cudaStream_t st) {
  d.alloc(std::max<size_t>(h.size(), 1));
  if (!h.empty()) NB_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
}

}  // namespace

struct nomad_b200_trainer {
  nomad_b200_ctx* ctx = nullptr;
  nomad_b200_train_config cfg{};
  uint64_t n = 0, C = 0, k = 0, kpad = 0, s = 0;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  uint32_t W = 0, w0 = 0, nwl = 0;
  double lr0 = 0.0;
  bool uniform_k = true;

  std::vector<uint32_t> sizes, c2w, orig_of;
  std::vector<WorkerDev> wk;
  std::vector<LocalCluster> lcl;
  std::vector<uint32_t> elig_h, pool_h, pool_off;
  std::vector<uint32_t> ell_h;
  std::vector<uint8_t> ncnt_h;
  std::vector<std::mt19937_64> rng;
  uint32_t max_slots = 0;
  size_t smem_replay = 0, smem_hog = 0;
  uint32_t hog_cells = 0;  // capacity of the hogwild kernel's shared cell table
  uint32_t replay_k = 0;   // replay: CTAs per worker
  DBuf<uint32_t> replay_bar;
  uint32_t hog_blocks = 0, chunk_heads = 0, total_chunks = 0, hog_wave = 1;
  DBuf<uint2> chunk_map;  // hogwild chunk -> (local worker, chunk within the worker)
  DBuf<uint32_t> chunk_counter;

  DBuf<double2> pos, means;
  DBuf<uint32_t> ell, elig, remote_ids, orig_of_d, cl_of, slot_gid, chunk_off;
  DBuf<uint8_t> ncnt;
  DBuf<double> wtab, remote_probs, cell_probs, slot, recv, sums, loss_acc;
  DBuf<unsigned long long> edge_acc, diverge;
  DBuf<WorkerDev> wk_d;
  DBuf<LocalCluster> lcl_d;
  uint32_t nchunks = 0, chunk = 4096;
  // replay tape
  DBuf<uint32_t> tape_head, tape_tails, tape_t, lvl_off, wk_lvl_base, wk_nlev, wk_draw_base;
  DBuf<double> loss_slot, wloss;
  std::vector<uint32_t> draw_base_h;

  uint64_t epochs_done = 0, edge_updates = 0;
  // device-side timing of the SGD kernel and the means+exchange step (CUDA
  // events on the launching stream), accumulated over all epochs run.
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  double sgd_ms = 0.0, means_ms = 0.0;
  uint64_t timed_epochs = 0;
  uint64_t comm_epochs = 0, comm_msgs = 0, comm_doubles = 0, comm_counts = 0;

  cudaStream_t st() const { return ctx->stream; }
  void launched(const char* name) { note_launch(ctx, name); }
  ~nomad_b200_trainer() {
    if (comm) ncclCommDestroy(comm);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }

  void validate() {
    // optimizer.hpp:63-71
    if (cfg.workers < 1) fail(kParameter, "workers must be >= 1");
    if (cfg.k < 1) fail(kParameter, "k must be >= 1");
    if (cfg.negatives < 1) fail(kParameter, "negatives must be >= 1");
    if (cfg.local_draws < 1) fail(kParameter, "local draws must be >= 1");
    if (cfg.batch_size < 1) fail(kParameter, "batch size must be >= 1");
    if (cfg.n_clusters != 0 && cfg.n_clusters < cfg.workers)
      fail(kParameter, "clusters must be >= workers");
    if (cfg.sgd_mode != NOMAD_B200_SGD_REPLAY && cfg.sgd_mode != NOMAD_B200_SGD_HOGWILD)
      fail(kParameter, "unknown sgd_mode");
    if (world < 1 || rank < 0 || rank >= world) fail(kParameter, "bad rank / world_size");
    if (cfg.workers % (uint64_t)world != 0)
      fail(kParameter, "workers must be a multiple of world_size");
  }

  // ---------------------------------------------------------------- setup
  void setup(const nomad_b200_graph* g, const nomad_b200_clusters* cl, const double* init,
             int init_loc, const void* nccl_id) {
    validate();
    n = cl->rows;
    C = cl->n_clusters;
    k = cfg.k;
    s = cfg.local_draws;
    W = (uint32_t)cfg.workers;
    if (g->rows != n) fail(kDimension, "graph and clusters cover different point counts");
    if (g->k != k) fail(kParameter, "graph k differs from config k");
    if (n >= 0xFFFFFFFFull) fail(kSize, "point ids are u32 (n < 2^32)");
    if (C < 1) fail(kParameter, "n_clusters must be >= 1");
    kpad = std::max<uint64_t>(16, (k + 15) / 16 * 16);
    if (k > 64) fail(kParameter, "k > 64 is not supported");
    if (s > 16) fail(kParameter, "local_draws > 16 is not supported");
    lr0 = cfg.lr0 > 0.0 ? cfg.lr0 : static_cast<double>(n) / 10.0;  // optimizer.hpp:79-81

    // host copies of assignment + offsets
    std::vector<uint32_t> assign(n), offs(n + 1);
    auto fetch = [&](std::vector<uint32_t>& dst, const uint32_t* src, size_t cnt, int loc) {
      NB_CUDA(cudaMemcpy(dst.data(), src, cnt * 4,
                         loc == NOMAD_B200_DEVICE ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
    };
    fetch(assign, cl->assignment, n, cl->location);
    fetch(offs, g->offsets, n + 1, g->location);
    sizes.assign(C, 0);
    for (uint64_t i = 0; i < n; ++i) {
      if (assign[i] >= C) fail(kParameter, "assignment entry out of range");
      ++sizes[assign[i]];
    }
    for (uint64_t r = 0; r < C; ++r)
      if (sizes[r] == 0) fail(kInternal, "empty cluster in means gather");

    // shard_clusters (optimizer.hpp:106-144) + rank / slot layout (plan.cu)
    ShardPlan plan = make_plan(sizes, W, world);
    c2w = plan.c2w;
    const auto& wclusters = plan.wclusters;

    nwl = W / world;
    w0 = rank * nwl;
    // members per cluster, ascending original id
    std::vector<uint64_t> cstart(C + 1, 0);
    for (uint64_t i = 0; i < n; ++i) ++cstart[assign[i] + 1];
    for (uint64_t r = 0; r < C; ++r) cstart[r + 1] += cstart[r];
    std::vector<uint32_t> members(n);
    {
      std::vector<uint64_t> f(cstart.begin(), cstart.end() - 1);
      for (uint64_t i = 0; i < n; ++i) members[f[assign[i]]++] = (uint32_t)i;
    }
    // local numbering
    std::vector<uint32_t> new_of(n, 0xFFFFFFFFu);
    orig_of.clear();
    wk.assign(nwl, WorkerDev{});
    lcl.clear();
    std::vector<uint32_t> cl_of_h;
    for (uint32_t wl = 0; wl < nwl; ++wl) {
      const uint32_t w = w0 + wl;
      WorkerDev& d = wk[wl];
      d.id = w;
      d.pstart = (uint32_t)orig_of.size();
      for (uint32_t c : wclusters[w]) {
        lcl.push_back(LocalCluster{(uint32_t)orig_of.size(), sizes[c], c, wl});
        for (uint64_t m = cstart[c]; m < cstart[c + 1]; ++m) {
          new_of[members[m]] = (uint32_t)orig_of.size();
          orig_of.push_back(members[m]);
          cl_of_h.push_back((uint32_t)lcl.size() - 1);
        }
      }
      d.npts = (uint32_t)orig_of.size() - d.pstart;
    }
    const uint64_t n_loc = orig_of.size();
    // per worker: pool (ascending original id) and eligible heads
    std::vector<std::vector<uint32_t>> pools(nwl), eligs(nwl);
    for (uint64_t i = 0; i < n; ++i) {
      const uint32_t w = c2w[assign[i]];
      if (w < w0 || w >= w0 + nwl) continue;
      pools[w - w0].push_back(new_of[i]);
      if (offs[i + 1] > offs[i]) eligs[w - w0].push_back(new_of[i]);
    }
    pool_h.clear();
    pool_off.assign(nwl + 1, 0);
    elig_h.clear();
    std::vector<uint32_t> rem_ids;
    std::vector<double> rem_probs;
    uint64_t total_elig = 0;
    uint32_t max_rem = 0;
    for (uint32_t wl = 0; wl < nwl; ++wl) {
      WorkerDev& d = wk[wl];
      pool_off[wl] = (uint32_t)pool_h.size();
      pool_h.insert(pool_h.end(), pools[wl].begin(), pools[wl].end());
      d.elig_off = (uint32_t)elig_h.size();
      d.n_elig = (uint32_t)eligs[wl].size();
      d.draws = d.n_elig;
      elig_h.insert(elig_h.end(), eligs[wl].begin(), eligs[wl].end());
      total_elig += d.n_elig;
      d.rem_off = (uint32_t)rem_ids.size();
      uint64_t remote = 0;
      for (uint64_t r = 0; r < C; ++r) {
        if (c2w[r] == d.id) continue;
        rem_ids.push_back((uint32_t)r);
        rem_probs.push_back(static_cast<double>(sizes[r]) / static_cast<double>(n));
        remote += sizes[r];
      }
      d.n_rem = (uint32_t)rem_ids.size() - d.rem_off;
      max_rem = std::max(max_rem, d.n_rem);
      d.local_mass = static_cast<double>(n - remote) / static_cast<double>(n);
    }
    pool_off[nwl] = (uint32_t)pool_h.size();
    // fit() fails when no point in the whole graph has a neighbour
    {
      uint64_t any = 0;
      for (uint64_t i = 0; i < n && !any; ++i) any = offs[i + 1] > offs[i];
      if (!any) fail(kConfig, "no point has any neighbor; nothing to train on");
    }
    (void)total_elig;

    // weights table (affinity.hpp:65-84: one table per neighbour count)
    std::vector<double> wt((k + 1) * k, 0.0);
    for (uint64_t c = 1; c <= k; ++c) {
      auto w = inverse_rank_weights(c);
      std::copy(w.begin(), w.end(), wt.begin() + c * k);
    }
    std::vector<double> cp(C);
    for (uint64_t r = 0; r < C; ++r) cp[r] = static_cast<double>(sizes[r]) / static_cast<double>(n);

    // ---- device state
    cudaStream_t S = st();
    upload(wtab, wt, S);
    upload(cell_probs, cp, S);
    upload(remote_ids, rem_ids, S);
    upload(remote_probs, rem_probs, S);
    upload(elig, elig_h, S);
    upload(orig_of_d, orig_of, S);
    upload(cl_of, cl_of_h, S);
    upload(lcl_d, lcl, S);
    // graph -> local ELL on the device
    {
      DBuf<uint32_t> off_tmp, nb_tmp, new_of_d;
      const uint32_t* off_p = g->offsets;
      const uint32_t* nb_p = g->neighbors;
      if (g->location != NOMAD_B200_DEVICE) {
        upload(off_tmp, offs, S);
        off_p = off_tmp.p;
        nb_tmp.alloc(std::max<uint64_t>(offs[n], 1));
        if (offs[n])
          NB_CUDA(cudaMemcpyAsync(nb_tmp.p, g->neighbors, (size_t)offs[n] * 4,
                                  cudaMemcpyHostToDevice, S));
        nb_p = nb_tmp.p;
      }
      upload(new_of_d, new_of, S);
      ell.alloc(std::max<uint64_t>(n_loc * kpad, 1));
      ncnt.alloc(std::max<uint64_t>(n_loc, 1));
      diverge.alloc(1);
      NB_CUDA(cudaMemsetAsync(diverge.p, 0xFF, 8, S));
      if (n_loc) {
        launch_build_ell(off_p, nb_p, orig_of_d.p, new_of_d.p, (uint32_t)n_loc, (uint32_t)kpad,
                         ell.p, ncnt.p, diverge.p, S);
        launched("k_build_ell");
      }
      unsigned long long bad = 0;
      NB_CUDA(cudaMemcpyAsync(&bad, diverge.p, 8, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
      if (bad != ~0ull) fail(kInternal, "kNN edge crosses shards or exceeds k (local point " +
                                            std::to_string(bad) + ")");
    }
    uniform_k = true;
    for (uint64_t i = 0; i < n; ++i)
      if (new_of[i] != 0xFFFFFFFFu && offs[i + 1] - offs[i] != k) { uniform_k = false; break; }
    if (cfg.sgd_mode == NOMAD_B200_SGD_REPLAY) {
      ell_h.resize(n_loc * kpad);
      ncnt_h.resize(n_loc);
      if (n_loc) {
        NB_CUDA(cudaMemcpy(ell_h.data(), ell.p, n_loc * kpad * 4, cudaMemcpyDeviceToHost));
        NB_CUDA(cudaMemcpy(ncnt_h.data(), ncnt.p, n_loc, cudaMemcpyDeviceToHost));
      }
      rng.clear();
      for (uint32_t wl = 0; wl < nwl; ++wl)  // optimizer.hpp:211-213, :371
        rng.emplace_back(stream_seed(cfg.seed, 0x776f726bull + wk[wl].id));
    }
    // positions in local order
    pos.alloc(std::max<uint64_t>(n_loc, 1));
    {
      DBuf<double> tmp;
      const double* src = init;
      if (init_loc != NOMAD_B200_DEVICE) {
        tmp.alloc(2 * n);
        NB_CUDA(cudaMemcpyAsync(tmp.p, init, n * 16, cudaMemcpyHostToDevice, S));
        src = tmp.p;
      }
      if (n_loc) {
        launch_gather_layout(reinterpret_cast<const double2*>(src), orig_of_d.p, (uint32_t)n_loc,
                             pos.p, S);
        launched("k_gather_layout");
      }
      NB_CUDA(cudaStreamSynchronize(S));
    }
    // means exchange: fixed slots per rank, static slot -> cluster map
    max_slots = plan.max_slots;
    const std::vector<uint32_t>& sg = plan.slot_cluster;
    upload(slot_gid, std::vector<uint32_t>(sg), S);
    slot.alloc(2 * (size_t)max_slots);
    NB_CUDA(cudaMemsetAsync(slot.p, 0, slot.bytes(), S));
    recv.alloc(2 * (size_t)world * max_slots);
    means.alloc(C);
    sums.alloc(2 * std::max<size_t>(lcl.size(), 1));
    NB_CUDA(cudaMemsetAsync(sums.p, 0, sums.bytes(), S));
    std::vector<uint32_t> co(lcl.size() + 1, 0);
    for (size_t c = 0; c < lcl.size(); ++c)
      co[c + 1] = co[c] + std::max<uint32_t>(1, (lcl[c].count + chunk - 1) / chunk);
    nchunks = co.back();
    upload(chunk_off, co, S);
    loss_acc.alloc(std::max<uint32_t>(nwl, 1));
    edge_acc.alloc(std::max<uint32_t>(nwl, 1));
    wloss.alloc(std::max<uint32_t>(nwl, 1));
    if (world > 1) {
      if (!nccl_id) fail(kParameter, "nccl_id required when world_size > 1");
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof id);
      NB_NCCL(ncclCommInitRank(&comm, world, id, rank));
    }

    // shared-memory budgets
    smem_replay = ((k + 1) * k + 3 * C) * sizeof(double);
    hog_cells = (uint32_t)(cfg.approx_all_but_own ? C : max_rem);
    smem_hog = ((((k + 1) * k + 1) & ~1ull) + 3 * (uint64_t)hog_cells) * sizeof(double);
    if (smem_replay > 200 * 1024 || smem_hog > 200 * 1024)
      fail(kSize, "too many clusters for the shared-memory cell table (C=" + std::to_string(C) + ")");
    // hogwild grid: per worker share of the resident capacity, capped by
    // npts / cap heads in flight
    if (cfg.sgd_mode == NOMAD_B200_SGD_HOGWILD) plan_hogwild_grid();
    upload(wk_d, wk, S);

    // epoch-0 means of the init layout (optimizer.hpp:384)
    compute_means_and_exchange();
    NB_CUDA(cudaStreamSynchronize(S));
    check_divergence(0, false);
  }

  void plan_hogwild_grid() {
    // Heads in flight on one shard <= shard size / cap,
    // never more blocks than are resident at once (the kernel pulls chunks
    // dynamically, so extra blocks would only idle). Chunks are ordered in
    // waves of `wave` shards, round-robin inside a wave: one shard at a time
    // keeps its positions L2-resident (config C), several at a time fill the
    // GPU when one shard's cap cannot (small shards, config B).
    const uint32_t cap = cfg.hogwild_cap ? cfg.hogwild_cap : 16;
    const uint32_t G = hogwild_group_size((uint32_t)kpad, (uint32_t)s);
    const uint64_t resident = hogwild_resident_blocks((uint32_t)kpad, (uint32_t)s, smem_hog, ctx->sm_count);
    uint64_t min_pts = ~0ull;
    for (auto& d : wk)
      if (d.draws) min_pts = std::min<uint64_t>(min_pts, d.npts);
    if (min_pts == ~0ull) min_pts = 1;
    const uint64_t heads_per_block = 256 / G;
    const uint64_t by_cap = std::max<uint64_t>(1, (min_pts / cap + heads_per_block - 1) / heads_per_block);
    uint32_t nact = 0;
    for (auto& d : wk) nact += d.draws ? 1u : 0u;
    const uint32_t wave = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>(std::max<uint32_t>(nact, 1), (resident + by_cap - 1) / by_cap));
    hog_blocks = (uint32_t)std::min<uint64_t>(resident, by_cap * wave);
    chunk_heads = (uint32_t)(heads_per_block * hogwild_chunk_rounds());
    std::vector<uint32_t> nchunk(nwl);
    for (uint32_t wl = 0; wl < nwl; ++wl) {
      WorkerDev& d = wk[wl];
      d.all_elig = d.n_elig == d.npts ? 1u : 0u;
      nchunk[wl] = (d.draws + chunk_heads - 1) / chunk_heads;
    }
    std::vector<uint2> cmap;
    for (uint32_t w0 = 0; w0 < nwl; w0 += wave) {
      const uint32_t w1 = std::min<uint32_t>(nwl, w0 + wave);
      uint32_t maxc = 0;
      for (uint32_t wl = w0; wl < w1; ++wl) maxc = std::max(maxc, nchunk[wl]);
      for (uint32_t lc = 0; lc < maxc; ++lc)
        for (uint32_t wl = w0; wl < w1; ++wl)
          if (lc < nchunk[wl]) cmap.push_back(make_uint2(wl, lc));
    }
    total_chunks = (uint32_t)cmap.size();
    hog_wave = wave;
    upload(chunk_map, cmap, st());
    chunk_counter.alloc(1);
    if (total_chunks == 0) hog_blocks = 0;
  }

  unsigned long long div_tag = 0;  // run-relative epoch tag of divergence keys (hogwild)
  // The throughput kernel's position rows are double-float while a run is in
  // progress (cfg.hogwild_double_float); outside run() they are f64 again.
  bool pos_is_df = false;
  void pos_format(bool df) {
    if (df == pos_is_df || !cfg.hogwild_double_float) return;
    launch_pos_df(pos.p, (uint32_t)orig_of.size(), df, st());
    launched("k_pos_df");
    pos_is_df = df;
  }

  void compute_means_and_exchange() {
    cudaStream_t S = st();
    const uint32_t ncl = (uint32_t)lcl.size();
    if (ncl) {
      if (cfg.sgd_mode == NOMAD_B200_SGD_REPLAY) {
        launch_means_exact(pos.p, lcl_d.p, ncl, slot.p, S);
        launched("k_means_exact");
      } else {
        launch_means_chunk(pos.p, pos_is_df, lcl_d.p, ncl, chunk, chunk_off.p, nchunks, sums.p,
                           diverge.p, div_tag, S);
        launched("k_means_chunk");
        launch_means_finalize(sums.p, lcl_d.p, ncl, slot.p, S);
        launched("k_means_finalize");
      }
    }
    const double* src = slot.p;
    if (world > 1) {
      NB_NCCL(ncclAllGather(slot.p, recv.p, 2 * (size_t)max_slots, ncclDouble, comm, S));
      src = recv.p;
    }
    launch_means_unpack(src, slot_gid.p, (uint32_t)world * max_slots, means.p, S);
    launched("k_means_unpack");
  }

  void check_divergence(uint64_t epoch, bool replay_key) {
    unsigned long long key = 0;
    NB_CUDA(cudaMemcpyAsync(&key, diverge.p, 8, cudaMemcpyDeviceToHost, st()));
    NB_CUDA(cudaStreamSynchronize(st()));
    if (key == ~0ull) return;
    char m[200];
    if (replay_key) {
      const uint64_t stride = 2 + k + s;
      const uint64_t t = (key >> 32) / stride;
      const uint32_t p = orig_of[(uint32_t)key];
      snprintf(m, sizeof m, "positions diverged at epoch %llu, head draw %llu (point %u)",
               (unsigned long long)epoch, (unsigned long long)t, p);
    } else {
      snprintf(m, sizeof m, "positions diverged at epoch %llu (point %u)",
               (unsigned long long)epoch, orig_of[(uint32_t)key]);
    }
    fail(kDivergence, m);
  }

  SgdParams params(double step, uint64_t epoch) {
    SgdParams P{};
    P.pos = pos.p;
    P.ell = ell.p;
    P.ncnt = uniform_k ? nullptr : ncnt.p;
    P.wtab = wtab.p;
    P.elig = elig.p;
    P.workers = wk_d.p;
    P.means = means.p;
    P.remote_ids = remote_ids.p;
    P.remote_probs = remote_probs.p;
    P.cl_of = cl_of.p;
    P.lclusters = lcl_d.p;
    P.cell_probs = cell_probs.p;
    P.loss_acc = loss_acc.p;
    P.edge_acc = edge_acc.p;
    P.diverge = diverge.p;
    P.n_workers = nwl;
    P.kpad = (uint32_t)kpad;
    P.k = (uint32_t)k;
    P.s = (uint32_t)s;
    P.m_total = (uint32_t)cfg.negatives;
    P.n_clusters = (uint32_t)C;
    P.head_only = cfg.head_only;
    P.double_float = cfg.hogwild_double_float ? 1 : 0;
    P.max_cells = hog_cells;
    P.all_but_own = cfg.approx_all_but_own;
    P.step = step;
    P.epoch = epoch;
    const uint64_t sk = mix_seed(cfg.seed ^ 0x686f67776c64ull);
    P.seed_lo = (uint32_t)sk;
    P.seed_hi = (uint32_t)(sk >> 32);
    P.chunk_counter = chunk_counter.p;
    P.total_chunks = total_chunks;
    P.chunk_heads = chunk_heads;
    P.chunk_map = chunk_map.p;
    return P;
  }

  // ------------------------------------------------------- replay tapes
  // For each local worker: the reference's draw sequence for this epoch
  // (optimizer.hpp:252-285) and its wavefront levels.
  // One epoch's replay tape: every worker's draws (mt19937_64 stream, the
  // reference's order) grouped by conflict level, worker-major.
  struct Tape {
    std::vector<uint32_t> th, tt, tid, loff, lbase, nlev;
    uint64_t edges = 0;
  };

  // Workers draw from their own streams and touch disjoint points, so their
  // tapes are built concurrently (one host thread per worker, up to the
  // hardware threads) straight into their slices of the epoch tape.
  void build_tapes(Tape& T) {
    std::vector<size_t> base(nwl + 1, 0);
    for (uint32_t wl = 0; wl < nwl; ++wl) base[wl + 1] = base[wl] + wk[wl].draws;
    T.th.resize(base[nwl]);
    T.tt.resize(base[nwl] * s);
    T.tid.resize(base[nwl]);
    std::vector<std::vector<uint32_t>> loffw(nwl);
    std::vector<uint32_t> maxl(nwl, 0);
    std::vector<uint64_t> edg(nwl, 0);
    auto one = [&](uint32_t wl) {
      const WorkerDev& d = wk[wl];
      const uint32_t D = d.draws;
      std::vector<uint32_t> head(D), tails((size_t)D * s), lev(D);
      uint32_t maxlev = 0;
      uint64_t edges = 0;
      auto& g = rng[wl];
      const uint32_t* pool = pool_h.data() + pool_off[wl];
      // pass 1: the stream's draws (optimizer.hpp:254-255, :284-285)
      for (uint32_t t = 0; t < D; ++t) {
        const uint32_t h = elig_h[d.elig_off + uniform_index(g, d.n_elig)];
        head[t] = h;
        uint32_t p0 = 0, pn = d.npts;
        if (cfg.approx_all_but_own) {
          // pool = own cluster members, ascending id == contiguous local ids
          const uint32_t c = local_cluster_of(h);
          p0 = lcl[c].start;
          pn = lcl[c].count;
          for (uint64_t q = 0; q < s; ++q) tails[(size_t)t * s + q] = p0 + (uint32_t)uniform_index(g, pn);
        } else {
          for (uint64_t q = 0; q < s; ++q) tails[(size_t)t * s + q] = pool[uniform_index(g, pn)];
        }
      }
      // pass 2: conflict levels over the worker's own point range (u16
      // levels, 2 bytes per point, while they fit; u32 otherwise), with the
      // neighbour rows of draws ahead prefetched
      const uint32_t p0w = d.pstart;
      auto levels = [&](auto& last) -> bool {
        using LT = typename std::decay_t<decltype(last)>::value_type;
        constexpr uint32_t AHEAD = 16;
        maxlev = 0;
        edges = 0;
        for (uint32_t t = 0; t < std::min(D, AHEAD); ++t)
          __builtin_prefetch(ell_h.data() + (size_t)head[t] * kpad);
        for (uint32_t t = 0; t < D; ++t) {
          if (t + AHEAD < D) __builtin_prefetch(ell_h.data() + (size_t)head[t + AHEAD] * kpad);
          const uint32_t h = head[t];
          // level = 1 + max level of every point it reads or writes
          const uint32_t cnt = ncnt_h[h];
          const uint32_t* nb = ell_h.data() + (size_t)h * kpad;
          const uint32_t* tl = tails.data() + (size_t)t * s;
          uint32_t L = last[h - p0w];
          for (uint32_t j = 0; j < cnt; ++j) L = std::max<uint32_t>(L, last[nb[j] - p0w]);
          for (uint64_t q = 0; q < s; ++q) L = std::max<uint32_t>(L, last[tl[q] - p0w]);
          ++L;
          if (L > std::numeric_limits<LT>::max()) return false;
          last[h - p0w] = (LT)L;
          for (uint32_t j = 0; j < cnt; ++j) last[nb[j] - p0w] = (LT)L;
          for (uint64_t q = 0; q < s; ++q) last[tl[q] - p0w] = (LT)L;
          lev[t] = L - 1;
          maxlev = std::max(maxlev, L);
          edges += cnt + s;
        }
        return true;
      };
      {
        std::vector<uint16_t> l16(d.npts, 0);
        if (!levels(l16)) {
          std::vector<uint32_t> l32(d.npts, 0);
          levels(l32);
        }
      }
      // counting sort by level (stable in t)
      std::vector<uint32_t> cnt_l(maxlev + 1, 0);
      for (uint32_t t = 0; t < D; ++t) ++cnt_l[lev[t] + 1];
      for (uint32_t l = 0; l < maxlev; ++l) cnt_l[l + 1] += cnt_l[l];
      const size_t b0 = base[wl];
      auto& lo = loffw[wl];
      lo.resize(maxlev + 1);
      for (uint32_t l = 0; l <= maxlev; ++l) lo[l] = (uint32_t)(b0 + cnt_l[l]);
      std::vector<uint32_t> fill(cnt_l.begin(), cnt_l.end() - 1);
      for (uint32_t t = 0; t < D; ++t) {
        const size_t at = b0 + fill[lev[t]]++;
        T.th[at] = head[t];
        T.tid[at] = t;
        for (uint64_t q = 0; q < s; ++q) T.tt[at * s + q] = tails[(size_t)t * s + q];
      }
      maxl[wl] = maxlev;
      edg[wl] = edges;
    };
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const unsigned nth = std::min<unsigned>(nwl, hw);
    if (nth <= 1) {
      for (uint32_t wl = 0; wl < nwl; ++wl) one(wl);
    } else {
      std::atomic<uint32_t> next{0};
      std::vector<std::thread> pool_t;
      for (unsigned i = 0; i < nth; ++i)
        pool_t.emplace_back([&] {
          for (uint32_t wl; (wl = next.fetch_add(1)) < nwl;) one(wl);
        });
      for (auto& x : pool_t) x.join();
    }
    T.loff.clear();
    T.lbase.assign(nwl, 0);
    T.nlev.assign(nwl, 0);
    T.edges = 0;
    for (uint32_t wl = 0; wl < nwl; ++wl) {
      T.lbase[wl] = (uint32_t)T.loff.size();
      T.nlev[wl] = maxl[wl];
      T.loff.insert(T.loff.end(), loffw[wl].begin(), loffw[wl].end());
      T.edges += edg[wl];
    }
  }

  // Continue the schedule at epoch `e` (resume from a checkpoint layout).
  // Throughput mode: draws are keyed by (seed, epoch, worker, t), nothing to
  // replay. Replay mode: each worker's mt19937_64 stream is advanced past the
  // skipped epochs' draws exactly as build_tapes consumes them.
  void seek(uint64_t e) {
    if (e > cfg.epochs) fail(kParameter, "epoch out of range for schedule");
    if (cfg.sgd_mode == NOMAD_B200_SGD_REPLAY) {
      if (e < epochs_done) fail(kParameter, "replay mode cannot seek backwards");
      for (; epochs_done < e; ++epochs_done)
        for (uint32_t wl = 0; wl < nwl; ++wl) {
          const WorkerDev& d = wk[wl];
          auto& g = rng[wl];
          for (uint32_t t = 0; t < d.draws; ++t) {
            const uint32_t h = elig_h[d.elig_off + uniform_index(g, d.n_elig)];
            const uint64_t pn = cfg.approx_all_but_own ? lcl[local_cluster_of(h)].count : d.npts;
            for (uint64_t q = 0; q < s; ++q) (void)uniform_index(g, pn);
          }
        }
    }
    epochs_done = e;
  }

  uint32_t local_cluster_of(uint32_t local_id) const {
    // lcl is sorted by start
    uint32_t lo = 0, hi = (uint32_t)lcl.size();
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) / 2;
      if (lcl[mid].start <= local_id) lo = mid; else hi = mid;
    }
    return lo;
  }

  // ---------------------------------------------------------------- run
  // Throughput mode without per-epoch host round trips: every epoch's SGD
  // kernel, means pass and all-gather are queued back to back; per-epoch
  // loss / edge sums land in device arrays and are read (and, multi-rank,
  // gathered) once at the end; divergence keys carry the epoch.
  void run_async(uint64_t n_epochs, double* epoch_loss) {
    cudaStream_t S = st();
    if (epochs_done + n_epochs > cfg.epochs) fail(kParameter, "epoch out of range for schedule");
    const uint64_t E = n_epochs, L = std::max<uint32_t>(nwl, 1);
    DBuf<double> lossb(E * L);
    DBuf<unsigned long long> edgeb(E * L);
    NB_CUDA(cudaMemsetAsync(lossb.p, 0, lossb.bytes(), S));
    NB_CUDA(cudaMemsetAsync(edgeb.p, 0, edgeb.bytes(), S));
    std::vector<cudaEvent_t> evs(3 * E);
    for (auto& x : evs) NB_CUDA(cudaEventCreate(&x));
    const uint64_t e_first = epochs_done;
    pos_format(true);
    for (uint64_t it = 0; it < E; ++it) {
      const uint64_t e = epochs_done;
      const double lr = lr0 * (1.0 - static_cast<double>(e) / static_cast<double>(cfg.epochs));
      const double step = lr / static_cast<double>(cfg.batch_size);
      SgdParams P = params(step, e);
      P.loss_acc = lossb.p + it * L;
      P.edge_acc = edgeb.p + it * L;
      NB_CUDA(cudaMemsetAsync(chunk_counter.p, 0, 4, S));
      NB_CUDA(cudaEventRecord(evs[3 * it], S));
      if (hog_blocks) {
        launch_sgd_hogwild(P, hog_blocks, smem_hog, S);
        launched("k_sgd_hogwild");
      }
      NB_CUDA(cudaEventRecord(evs[3 * it + 1], S));
      div_tag = it;
      compute_means_and_exchange();
      NB_CUDA(cudaEventRecord(evs[3 * it + 2], S));
      ++comm_epochs;
      comm_msgs += W;
      comm_doubles += 2 * C;
      comm_counts += C;
      ++epochs_done;
    }
    div_tag = 0;
    pos_format(false);
    std::vector<double> lh(E * L);
    std::vector<unsigned long long> eh(E * L);
    NB_CUDA(cudaMemcpyAsync(lh.data(), lossb.p, E * L * 8, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaMemcpyAsync(eh.data(), edgeb.p, E * L * 8, cudaMemcpyDeviceToHost, S));
    std::vector<double> all;
    if (world > 1) {
      DBuf<double> g((size_t)world * E * L);
      NB_NCCL(ncclAllGather(lossb.p, g.p, E * L, ncclDouble, comm, S));
      all.resize((size_t)world * E * L);
      NB_CUDA(cudaMemcpyAsync(all.data(), g.p, all.size() * 8, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
    }
    unsigned long long key = 0;
    NB_CUDA(cudaMemcpyAsync(&key, diverge.p, 8, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    for (uint64_t it = 0; it < E; ++it) {
      float a = 0.f, b = 0.f;
      NB_CUDA(cudaEventElapsedTime(&a, evs[3 * it], evs[3 * it + 1]));
      NB_CUDA(cudaEventElapsedTime(&b, evs[3 * it + 1], evs[3 * it + 2]));
      sgd_ms += a;
      means_ms += b;
      ++timed_epochs;
    }
    for (auto& x : evs) cudaEventDestroy(x);
    if (key != ~0ull) {
      char m[200];
      snprintf(m, sizeof m, "positions diverged at epoch %llu (point %u)",
               (unsigned long long)(e_first + (key >> 32)), orig_of[(uint32_t)key]);
      fail(kDivergence, m);
    }
    const uint64_t heads = world > 1 ? total_heads_global() : [&] {
      uint64_t h = 0;
      for (auto& d : wk) h += d.draws;
      return h;
    }();
    for (uint64_t it = 0; it < E; ++it) {
      double loss_sum = 0.0;  // worker order: rank-major, then local worker
      if (world > 1) {
        for (int r = 0; r < world; ++r)
          for (uint32_t wl = 0; wl < nwl; ++wl) loss_sum += all[((size_t)r * E + it) * L + wl];
      } else {
        for (uint32_t wl = 0; wl < nwl; ++wl) loss_sum += lh[it * L + wl];
      }
      for (uint32_t wl = 0; wl < nwl; ++wl) edge_updates += eh[it * L + wl];
      if (epoch_loss) epoch_loss[it] = heads > 0 ? loss_sum / static_cast<double>(heads) : 0.0;
    }
  }

  void run(uint64_t n_epochs, double* epoch_loss) {
    if (cfg.sgd_mode == NOMAD_B200_SGD_HOGWILD && !cfg.verbose) return run_async(n_epochs, epoch_loss);
    cudaStream_t S = st();
    if (draw_base_h.empty()) {
      draw_base_h.assign(nwl, 0);
      uint32_t acc = 0;
      for (uint32_t wl = 0; wl < nwl; ++wl) { draw_base_h[wl] = acc; acc += wk[wl].draws; }
      upload(wk_draw_base, draw_base_h, S);
      loss_slot.alloc(std::max<uint32_t>(acc, 1));
    }
    // replay: the next epoch's tape is built on host threads while this
    // epoch runs on the GPU (tapes depend only on the workers' streams);
    // only within this call, so the streams end exactly n_epochs ahead
    Tape cur, nxt;
    std::thread prefetch;
    struct Joiner {
      std::thread& t;
      ~Joiner() {
        if (t.joinable()) t.join();
      }
    } joiner{prefetch};
    const bool replay = cfg.sgd_mode == NOMAD_B200_SGD_REPLAY;
    std::vector<double> wl_loss(nwl), all_loss(world * std::max<uint32_t>(nwl, 1));
    std::vector<unsigned long long> wl_edges(nwl);
    DBuf<double> gl;  // gathered per-worker losses (multi-rank)
    DBuf<double> gheads;
    for (uint64_t it = 0; it < n_epochs; ++it) {
      const uint64_t e = epochs_done;
      if (e >= cfg.epochs) fail(kParameter, "epoch out of range for schedule");
      const auto t0 = std::chrono::steady_clock::now();
      // optimizer.hpp:85-91, :390-391
      const double lr = lr0 * (1.0 - static_cast<double>(e) / static_cast<double>(cfg.epochs));
      const double step = lr / static_cast<double>(cfg.batch_size);
      SgdParams P = params(step, e);
      uint64_t edges = 0;
      if (!ev[0])
        for (auto& x : ev) NB_CUDA(cudaEventCreate(&x));
      if (replay) {
        if (it == 0) {
          build_tapes(cur);
        } else {
          prefetch.join();
          std::swap(cur, nxt);
        }
        if (it + 1 < n_epochs) prefetch = std::thread([this, &nxt] { build_tapes(nxt); });
        edges = cur.edges;
        if (std::getenv("NOMAD_B200_DEBUG_REPLAY") && it == 0)
          for (uint32_t wl = 0; wl < nwl; ++wl)
            std::fprintf(stderr, "replay worker %u: %u draws, %u levels\n", wl, wk[wl].draws,
                         cur.nlev[wl]);
        upload(tape_head, cur.th, S);
        upload(tape_tails, cur.tt, S);
        upload(tape_t, cur.tid, S);
        upload(lvl_off, cur.loff, S);
        upload(wk_lvl_base, cur.lbase, S);
        upload(wk_nlev, cur.nlev, S);
        P.tape_head = tape_head.p;
        P.tape_tails = tape_tails.p;
        P.tape_t = tape_t.p;
        P.lvl_off = lvl_off.p;
        P.wk_lvl_base = wk_lvl_base.p;
        P.wk_nlev = wk_nlev.p;
        P.loss_slot = loss_slot.p;
        P.wk_draw_base = wk_draw_base.p;
        if (!replay_k) {
          replay_k = replay_ctas_per_worker(nwl, smem_replay, ctx->sm_count);
          replay_bar.alloc(std::max<uint32_t>(nwl, 1));
        }
        P.replay_ctas = replay_k;
        P.replay_bar = replay_bar.p;
        NB_CUDA(cudaEventRecord(ev[0], S));
        if (nwl) {
          launch_sgd_replay(P, nwl, smem_replay, S);
          launched("k_sgd_replay");
          launch_loss_seq(loss_slot.p, wk_draw_base.p, wk_d.p, nwl, wloss.p, S);
          launched("k_loss_seq");
        }
        NB_CUDA(cudaEventRecord(ev[1], S));
      } else {
        NB_CUDA(cudaMemsetAsync(loss_acc.p, 0, loss_acc.bytes(), S));
        NB_CUDA(cudaMemsetAsync(edge_acc.p, 0, edge_acc.bytes(), S));
        NB_CUDA(cudaMemsetAsync(chunk_counter.p, 0, 4, S));
        pos_format(true);
        NB_CUDA(cudaEventRecord(ev[0], S));
        if (hog_blocks) {
          launch_sgd_hogwild(P, hog_blocks, smem_hog, S);
          launched("k_sgd_hogwild");
        }
        NB_CUDA(cudaEventRecord(ev[1], S));
      }
      compute_means_and_exchange();
      pos_format(false);
      NB_CUDA(cudaEventRecord(ev[2], S));
      // per-worker loss sums -> epoch mean (optimizer.hpp:444-451)
      const double* lsrc = cfg.sgd_mode == NOMAD_B200_SGD_REPLAY ? wloss.p : loss_acc.p;
      if (nwl) NB_CUDA(cudaMemcpyAsync(wl_loss.data(), lsrc, nwl * 8, cudaMemcpyDeviceToHost, S));
      if (cfg.sgd_mode == NOMAD_B200_SGD_HOGWILD && nwl)
        NB_CUDA(cudaMemcpyAsync(wl_edges.data(), edge_acc.p, nwl * 8, cudaMemcpyDeviceToHost, S));
      if (world > 1) {
        if (!gl.p) { gl.alloc((size_t)world * nwl); }
        NB_NCCL(ncclAllGather(lsrc, gl.p, nwl, ncclDouble, comm, S));
        NB_CUDA(cudaMemcpyAsync(all_loss.data(), gl.p, (size_t)world * nwl * 8,
                                cudaMemcpyDeviceToHost, S));
      }
      check_divergence(e, cfg.sgd_mode == NOMAD_B200_SGD_REPLAY);  // syncs the stream
      {
        float a = 0.f, b = 0.f;
        NB_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
        NB_CUDA(cudaEventElapsedTime(&b, ev[1], ev[2]));
        sgd_ms += a;
        means_ms += b;
        ++timed_epochs;
      }
      if (cfg.sgd_mode == NOMAD_B200_SGD_HOGWILD)
        for (uint32_t wl = 0; wl < nwl; ++wl) edges += wl_edges[wl];
      edge_updates += edges;
      double loss_sum = 0.0;
      uint64_t heads = 0;
      if (world > 1) {
        for (size_t i = 0; i < all_loss.size(); ++i) loss_sum += all_loss[i];
        // every worker draws its eligible count (global, identical on ranks)
        heads = total_heads_global();
      } else {
        for (uint32_t wl = 0; wl < nwl; ++wl) { loss_sum += wl_loss[wl]; heads += wk[wl].draws; }
      }
      const double mean_loss = heads > 0 ? loss_sum / static_cast<double>(heads) : 0.0;
      if (epoch_loss) epoch_loss[it] = mean_loss;
      // CommLog: one message per worker (optimizer.hpp:429-440)
      ++comm_epochs;
      comm_msgs += W;
      comm_doubles += 2 * C;
      comm_counts += C;
      ++epochs_done;
      if (cfg.verbose) {
        const double secs =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "epoch %llu/%llu lr %.6g loss %.6f time %.2fs\n",
                     (unsigned long long)(e + 1), (unsigned long long)cfg.epochs, lr, mean_loss,
                     secs);
      }
    }
  }

  uint64_t global_heads = 0;
  uint64_t total_heads_global() {
    if (!global_heads) {
      // eligible counts of all workers: every rank knows the plan but only
      // its own eligibility; gather once.
      DBuf<double> a(1), b((size_t)world);
      double mine = 0;
      for (auto& d : wk) mine += d.draws;
      NB_CUDA(cudaMemcpy(a.p, &mine, 8, cudaMemcpyHostToDevice));
      NB_NCCL(ncclAllGather(a.p, b.p, 1, ncclDouble, comm, st()));
      std::vector<double> h(world);
      NB_CUDA(cudaMemcpyAsync(h.data(), b.p, world * 8, cudaMemcpyDeviceToHost, st()));
      NB_CUDA(cudaStreamSynchronize(st()));
      for (double v : h) global_heads += (uint64_t)v;
    }
    return global_heads;
  }

  // Replace the positions (original order, n x 2) and re-gather the means
  // snapshot, as if the epoch loop had been given this layout.
  DBuf<double2> stage;  // n rows, original order (host <-> device staging)

  void set_layout(const double* in, int loc) {
    cudaStream_t S = st();
    const uint32_t n_loc = (uint32_t)orig_of.size();
    const double* src = in;
    if (loc != NOMAD_B200_DEVICE) {
      if (stage.n != n) stage.alloc(n);
      NB_CUDA(cudaMemcpyAsync(stage.p, in, n * 16, cudaMemcpyHostToDevice, S));
      src = reinterpret_cast<const double*>(stage.p);
    }
    if (n_loc) {
      launch_gather_layout(reinterpret_cast<const double2*>(src), orig_of_d.p, n_loc, pos.p, S);
      launched("k_gather_layout");
    }
    compute_means_and_exchange();
    NB_CUDA(cudaStreamSynchronize(S));
  }

  void layout(double* out, int loc) {
    cudaStream_t S = st();
    const uint32_t n_loc = (uint32_t)orig_of.size();
    if (loc == NOMAD_B200_DEVICE) {
      if (n_loc) {
        launch_scatter_layout(pos.p, orig_of_d.p, n_loc, reinterpret_cast<double2*>(out), S);
        launched("k_scatter_layout");
      }
      NB_CUDA(cudaStreamSynchronize(S));
      return;
    }
    if (world == 1) {  // every row is local: scatter on the device, one D2H copy
      if (stage.n != n) stage.alloc(n);
      if (n_loc) {
        launch_scatter_layout(pos.p, orig_of_d.p, n_loc, stage.p, S);
        launched("k_scatter_layout");
      }
      NB_CUDA(cudaMemcpyAsync(out, stage.p, n * 16, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
      return;
    }
    std::vector<double> h(2 * (size_t)n_loc);
    if (n_loc) NB_CUDA(cudaMemcpyAsync(h.data(), pos.p, h.size() * 8, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    for (uint32_t i = 0; i < n_loc; ++i) {
      out[2 * (size_t)orig_of[i]] = h[2 * (size_t)i];
      out[2 * (size_t)orig_of[i] + 1] = h[2 * (size_t)i + 1];
    }
  }
};

extern "C" {

int32_t nomad_b200_trainer_create(nomad_b200_ctx* ctx, const nomad_b200_graph* graph,
                                  const nomad_b200_clusters* clusters, const double* init,
                                  int32_t init_loc, const nomad_b200_train_config* cfg,
                                  int32_t rank, int32_t world, const void* nccl_id,
                                  nomad_b200_trainer** out) {
  return guard([&] {
    if (!ctx || !graph || !clusters || !init || !cfg || !out) fail(kParameter, "NULL argument");
    bind_device(ctx);
    auto* t = new nomad_b200_trainer();
    t->ctx = ctx;
    t->cfg = *cfg;
    t->rank = rank;
    t->world = world;
    try {
      t->setup(graph, clusters, init, init_loc, nccl_id);
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

int32_t nomad_b200_trainer_destroy(nomad_b200_trainer* t) {
  return guard([&] {
    if (!t) return;
    bind_device(t->ctx);
    cudaStreamSynchronize(t->ctx->stream);
    delete t;
  });
}

int32_t nomad_b200_trainer_run(nomad_b200_trainer* t, uint64_t n_epochs, double* epoch_loss) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    bind_device(t->ctx);
    t->run(n_epochs, epoch_loss);
  });
}

int32_t nomad_b200_trainer_layout(nomad_b200_trainer* t, double* out, int32_t loc) {
  return guard([&] {
    if (!t || !out) fail(kParameter, "NULL argument");
    bind_device(t->ctx);
    t->layout(out, loc);
  });
}

int32_t nomad_b200_trainer_means(nomad_b200_trainer* t, double* means, uint32_t* counts) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    bind_device(t->ctx);
    if (means) {
      NB_CUDA(cudaMemcpyAsync(means, t->means.p, t->C * 16, cudaMemcpyDeviceToHost, t->st()));
      NB_CUDA(cudaStreamSynchronize(t->st()));
    }
    if (counts) std::memcpy(counts, t->sizes.data(), t->C * 4);
  });
}

int32_t nomad_b200_trainer_comm(nomad_b200_trainer* t, uint64_t* epochs, uint64_t* messages,
                                uint64_t* doubles, uint64_t* counts) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    if (epochs) *epochs = t->comm_epochs;
    if (messages) *messages = t->comm_msgs;
    if (doubles) *doubles = t->comm_doubles;
    if (counts) *counts = t->comm_counts;
  });
}

int32_t nomad_b200_trainer_set_layout(nomad_b200_trainer* t, const double* layout, int32_t loc) {
  return guard([&] {
    if (!t || !layout) fail(kParameter, "NULL argument");
    bind_device(t->ctx);
    t->set_layout(layout, loc);
  });
}

int32_t nomad_b200_trainer_timing(nomad_b200_trainer* t, double* sgd_ms, double* means_ms,
                                  uint64_t* epochs) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    if (sgd_ms) *sgd_ms = t->sgd_ms;
    if (means_ms) *means_ms = t->means_ms;
    if (epochs) *epochs = t->timed_epochs;
  });
}

int32_t nomad_b200_trainer_seek(nomad_b200_trainer* t, uint64_t epoch) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    t->seek(epoch);
  });
}

int32_t nomad_b200_trainer_progress(nomad_b200_trainer* t, uint64_t* epochs_done,
                                    uint64_t* edge_updates) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    if (epochs_done) *epochs_done = t->epochs_done;
    if (edge_updates) *edge_updates = t->edge_updates;
  });
}

}  // extern "C"
