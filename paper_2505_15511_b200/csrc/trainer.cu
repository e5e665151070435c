// Host orchestration of the epoch loop: the setup half of fit()
// (optimizer.hpp:342-386), the epoch loop (:388-470) and the cross-shard
// means all-gather (:411-442) over NCCL (one process per GPU, or one process
// driving a group of GPUs) or a loopback exchange (a group on one GPU). All
// numerics run in sgd.cu kernels; the host builds the shard plan / local
// numbering (O(n) integer work), and,
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
#include <memory>
#include <numeric>
#include <random>

#include "common.cuh"
#include "hostcopy.cuh"
#include "plan.cuh"
#include "replay.cuh"
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

template <class T>
void upload(DBuf<T>& d, const std::vector<T>& h, cudaStream_t st) {
  d.alloc(std::max<size_t>(h.size(), 1));
  if (!h.empty()) NB_CUDA(cudaMemcpyAsync(d.p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, st));
}

}  // namespace

namespace nb {

struct DivKey {
  uint64_t worker = ~0ull, key = ~0ull;
  bool operator<(const DivKey& o) const {
    return worker != o.worker ? worker < o.worker : key < o.key;
  }
  bool none() const { return key == ~0ull; }
};

// One rank's share of the epoch loop: the workers [rank*W/world,
// (rank+1)*W/world) on one context. A trainer object (below) drives one rank
// (one process per GPU, NCCL between processes) or all G ranks of a group
// (one process, NCCL between devices or a loopback exchange on one device).
// An epoch is split into phases so a group can interleave its ranks:
// launch (SGD + this rank's means into its slot) -> exchange -> finish
// (unpack the all-gathered means, results to host).
struct RankTrainer {
  nomad_b200_ctx* ctx = nullptr;
  nomad_b200_train_config cfg{};
  uint64_t n = 0, C = 0, k = 0, kpad = 0, s = 0;
  int rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  bool own_comm = false;
  bool grouped = false;  // the means exchange is driven by the group trainer
  uint32_t W = 0, w0 = 0, nwl = 0;
  double lr0 = 0.0;
  bool uniform_k = true;

  std::vector<uint32_t> sizes, c2w, orig_of;
  std::vector<WorkerDev> wk;
  std::vector<LocalCluster> lcl;
  std::vector<uint32_t> elig_h, pool_h, pool_off;
  // replay: the workers' std::mt19937_64 streams live on the device
  // (double-buffered epoch start / end states); host copies only for seek and
  // the rejection fallback
  DBuf<MtState> mt_a, mt_b;
  // the next epoch's words, formed on a side stream while this epoch's
  // dependency pass runs: words2 + the state after them (mt_c), valid for
  // epoch pre_epoch (prefetch off for ranks sharing a device: the dataflow
  // kernel needs every SM to itself)
  DBuf<MtState> mt_c;
  DBuf<unsigned long long> words2;
  bool prefetch = true, pre_ok = false;
  uint64_t pre_epoch = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t pre_ev = nullptr, map_ev = nullptr;
  DBuf<uint64_t> wcount, wbase;
  DBuf<unsigned long long> words, redges;
  DBuf<double2> rmbox;
  DBuf<uint2> rlink;
  DBuf<uint32_t> pool_d, pool_off_d, rheads, rtails, tkey, tval, tkey2, tval2, rpred, reject,
      ticket, pt_base, stall;
  DBuf<uint8_t> rdone, sort_tmp;
  size_t sort_bytes = 0;
  uint32_t df_blocks = 0, total_draws = 0, max_draws = 0;
  uint32_t max_slots = 0;
  size_t smem_replay = 0, smem_hog = 0;
  uint32_t hog_cells = 0;  // cells per worker of the hogwild cell table
  bool gcells = false;     // cell tables in global memory (too many clusters for shared memory)
  uint32_t hog_blocks = 0, chunk_heads = 0, total_chunks = 0, hog_wave = 1;
  DBuf<uint2> chunk_map;  // hogwild chunk -> (local worker, chunk within the worker)
  DBuf<uint32_t> chunk_counter;

  DBuf<double2> pos, means, gcell_mu;
  DBuf<uint32_t> ell, elig, remote_ids, orig_of_d, cl_of, slot_gid, chunk_off;
  DBuf<uint8_t> ncnt;
  DBuf<double> wtab, remote_probs, cell_probs, slot, recv, sums, loss_acc, gcell_w, cm3;
  DBuf<unsigned long long> edge_acc, diverge;
  DBuf<WorkerDev> wk_d;
  DBuf<LocalCluster> lcl_d;
  uint32_t nchunks = 0, chunk = 4096;
  DBuf<uint32_t> wk_draw_base;
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
  void bind() { bind_device(ctx); }
  void launched(const char* name) { note_launch(ctx, name); }
  ~RankTrainer() {
    if (side) {
      cudaStreamSynchronize(side);
      cudaStreamDestroy(side);
    }
    if (pre_ev) cudaEventDestroy(pre_ev);
    if (map_ev) cudaEventDestroy(map_ev);
    if (comm && own_comm) ncclCommDestroy(comm);
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
  // Everything but the epoch-0 means (the caller runs the first exchange).
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
    if (k > 64) fail(kParameter, "k > 64 is not supported");
    if (s > 16) fail(kParameter, "local_draws > 16 is not supported");
    // ELL row width = the throughput kernel's compiled neighbour capacity
    kpad = k <= 16 ? 16 : (k <= 32 ? 32 : 64);
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
    uint32_t max_rem = 0;
    for (uint32_t wl = 0; wl < nwl; ++wl) {
      WorkerDev& d = wk[wl];
      pool_off[wl] = (uint32_t)pool_h.size();
      pool_h.insert(pool_h.end(), pools[wl].begin(), pools[wl].end());
      d.elig_off = (uint32_t)elig_h.size();
      d.n_elig = (uint32_t)eligs[wl].size();
      d.draws = d.n_elig;
      elig_h.insert(elig_h.end(), eligs[wl].begin(), eligs[wl].end());
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

    // weights table (affinity.hpp:65-84: one table per neighbour count)
    const std::vector<double> wt = weight_table(k);
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
      diverge.alloc(std::max<uint32_t>(nwl, 1));
      NB_CUDA(cudaMemsetAsync(diverge.p, 0xFF, diverge.bytes(), S));
      if (n_loc) {
        launch_build_ell(off_p, nb_p, orig_of_d.p, new_of_d.p, cl_of.p, lcl_d.p, (uint32_t)n_loc,
                         (uint32_t)k, (uint32_t)kpad, ell.p, ncnt.p, diverge.p, S);
        launched("k_build_ell");
      }
      unsigned long long bad = 0;
      NB_CUDA(cudaMemcpyAsync(&bad, diverge.p, 8, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
      if (bad != ~0ull)
        fail(kParameter, "kNN list of point " + std::to_string(orig_of[(uint32_t)bad]) +
                             " is longer than k or names a point outside its worker's shard");
    }
    uniform_k = true;
    for (uint64_t i = 0; i < n; ++i)
      if (new_of[i] != 0xFFFFFFFFu && offs[i + 1] - offs[i] != k) { uniform_k = false; break; }
    if (cfg.sgd_mode == NOMAD_B200_SGD_REPLAY) setup_replay(cl_of_h);
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
    if (world > 1 && !grouped) {
      if (!nccl_id) fail(kParameter, "nccl_id required when world_size > 1");
      ncclUniqueId id;
      std::memcpy(&id, nccl_id, sizeof id);
      NB_NCCL(ncclCommInitRank(&comm, world, id, rank));
      own_comm = true;
    }

    // cell tables: shared memory while they fit (the headline configs), else
    // global memory read through L1 (the reference's auto C = ceil(n/4096)
    // has ~14.6k clusters at 60M rows, optimizer.hpp:73-77)
    const uint64_t wts = (((k + 1) * k) + 1) & ~1ull;
    hog_cells = (uint32_t)std::max<uint64_t>(cfg.approx_all_but_own ? C : max_rem, 1);
    if (cfg.sgd_mode == NOMAD_B200_SGD_REPLAY) {
      smem_replay = ((k + 1) * k + 3 * C) * sizeof(double);
      if (smem_replay > 96 * 1024) {
        gcells = true;
        smem_replay = (k + 1) * k * sizeof(double);
      }
    } else {
      smem_hog = (wts + 3 * (uint64_t)hog_cells) * sizeof(double);
      if (smem_hog > 48 * 1024) {
        gcells = true;
        smem_hog = wts * sizeof(double);
      }
    }
    if (gcells) {
      gcell_mu.alloc((size_t)std::max<uint32_t>(nwl, 1) * hog_cells);
      gcell_w.alloc((size_t)std::max<uint32_t>(nwl, 1) * hog_cells);
      cm3.alloc(3 * C);
    }
    // hogwild grid: per worker share of the resident capacity, capped by
    // npts / cap heads in flight
    if (cfg.sgd_mode == NOMAD_B200_SGD_HOGWILD) plan_hogwild_grid();
    upload(wk_d, wk, S);
  }

  // Device replay state: the workers' streams (optimizer.hpp:211-213, :371:
  // stream_seed(seed, "work" + worker id)), per-epoch draw / dependency
  // buffers sized for one epoch of every local worker.
  void setup_replay(const std::vector<uint32_t>& cl_of_h) {
    cudaStream_t S = st();
    std::vector<MtState> st0(std::max<uint32_t>(nwl, 1));
    for (uint32_t wl = 0; wl < nwl; ++wl) {
      Mt64 m;
      m.seed(stream_seed(cfg.seed, 0x776f726bull + wk[wl].id));
      st0[wl] = m.s;
    }
    upload(mt_a, st0, S);
    mt_b.alloc(st0.size());
    draw_base_h.assign(nwl, 0);
    std::vector<uint64_t> wc(std::max<uint32_t>(nwl, 1), 0), wb(std::max<uint32_t>(nwl, 1), 0);
    uint64_t acc = 0, wacc = 0;
    max_draws = 0;
    for (uint32_t wl = 0; wl < nwl; ++wl) {
      draw_base_h[wl] = (uint32_t)acc;
      wc[wl] = (uint64_t)wk[wl].draws * (1 + s);
      wb[wl] = wacc;
      acc += wk[wl].draws;
      wacc += wc[wl];
      max_draws = std::max(max_draws, wk[wl].draws);
    }
    if (acc >= 0xFFFFFFFFull) fail(kSize, "replay draws per rank exceed 2^32");
    total_draws = (uint32_t)acc;
    upload(wk_draw_base, draw_base_h, S);
    upload(wcount, wc, S);
    upload(wbase, wb, S);
    upload(pool_d, pool_h, S);
    upload(pool_off_d, pool_off, S);
    std::vector<uint32_t> ptb(orig_of.size());
    for (size_t v = 0; v < ptb.size(); ++v) ptb[v] = draw_base_h[lcl[cl_of_h[v]].worker];
    upload(pt_base, ptb, S);
    const uint64_t T = 1 + k + s, D = std::max<uint64_t>(acc, 1);
    words.alloc(std::max<uint64_t>(wacc, 1));
    rheads.alloc(D);
    rtails.alloc(D * s);
    if (D * T >= 0xFFFFFFFFull) fail(kSize, "replay touches per rank exceed 2^32");
    tkey.alloc(D * T);
    tval.alloc(D * T);
    tkey2.alloc(D * T);
    tval2.alloc(D * T);
    if (dataflow_warp_form((uint32_t)k, (uint32_t)s)) {  // position mailboxes (replay.cu)
      rlink.alloc(D * T);
      rmbox.alloc(D * T);
      // all empty; every mailbox is emptied again by its reader, so one fill lasts
      NB_CUDA(cudaMemsetAsync(rmbox.p, 0xFF, rmbox.bytes(), S));
    } else {
      rpred.alloc(D * T);
    }
    rdone.alloc(D);
    loss_slot.alloc(D);
    // (warp form: all-ones = not yet written; the loss followers empty each
    // slot again after reading it, so one fill lasts)
    NB_CUDA(cudaMemsetAsync(loss_slot.p, 0xFF, loss_slot.bytes(), S));
    reject.alloc(std::max<uint32_t>(nwl, 1));
    redges.alloc(std::max<uint32_t>(nwl, 1));
    ticket.alloc(1);
    stall.alloc(1);
    NB_CUDA(cudaMemsetAsync(stall.p, 0, 4, S));
    sort_bytes = replay_sort_bytes(D * T, (uint32_t)orig_of.size());
    sort_tmp.alloc(std::max<size_t>(sort_bytes, 1));
  }

  ReplayDev replay_dev() {
    ReplayDev R{};
    R.nwl = nwl;
    R.s = (uint32_t)s;
    R.T = (uint32_t)(1 + k + s);
    R.draw_base = wk_draw_base.p;
    R.word_base = wbase.p;
    R.st_in = mt_a.p;
    R.st_out = mt_b.p;
    R.words = words.p;
    R.heads = rheads.p;
    R.tails = rtails.p;
    R.tkey = tkey.p;
    R.tval = tval.p;
    R.tkey2 = tkey2.p;
    R.tval2 = tval2.p;
    R.pred = rpred.p;
    R.link = rlink.p;
    R.mbox = rmbox.p;
    R.n_loc = (uint32_t)orig_of.size();
    R.reject = reject.p;
    R.edges = redges.p;
    R.done = rdone.p;
    R.ticket = ticket.p;
    R.stall = stall.p;
    R.wloss = wloss.p;
    // loss followers (warp form), when the grid leaves room for them
    R.followers = 0;
    if (rlink.p && df_blocks) {
      const uint32_t f = std::min<uint32_t>(std::max<uint32_t>(nwl, 1), 32u);
      if ((uint64_t)df_blocks * 8 >= 8ull * f) R.followers = f;  // at most 1/8 of the warps
    }
    R.pt_base = pt_base.p;
    const uint32_t per = dataflow_draws_per_chunk((uint32_t)k, (uint32_t)s);
    R.total_chunks = nwl * ((max_draws + per - 1) / per);
    R.max_draws = max_draws;
    R.total_draws = total_draws;
    static const uint32_t nap = [] {
      const char* e = std::getenv("NOMAD_B200_DF_NAP");
      return e ? (uint32_t)std::max(1, std::atoi(e)) : 64u;
    }();
    R.nap_cap = nap;
    return R;
  }

  // A worker whose epoch hit the rejection branch of uniform_index
  // (rng.hpp:49-55, probability ~n / 2^64 per draw): its draws are made on
  // the host from the epoch's start state, consuming the extra words exactly
  // as the reference does (optimizer.hpp:254-255, :284-285).
  void host_draws(uint32_t wl) {
    cudaStream_t S = st();
    Mt64 m;
    NB_CUDA(cudaMemcpy(&m.s, mt_a.p + wl, sizeof(MtState), cudaMemcpyDeviceToHost));
    const WorkerDev& d = wk[wl];
    std::vector<uint32_t> hd(d.draws), tl((size_t)d.draws * s);
    for (uint32_t t = 0; t < d.draws; ++t) {
      const uint32_t h = elig_h[d.elig_off + m.uniform_index(d.n_elig)];
      hd[t] = h;
      if (cfg.approx_all_but_own) {
        const LocalCluster& L = lcl[local_cluster_of(h)];
        for (uint64_t q = 0; q < s; ++q) tl[(size_t)t * s + q] = L.start + (uint32_t)m.uniform_index(L.count);
      } else {
        const uint32_t* pool = pool_h.data() + pool_off[wl];
        for (uint64_t q = 0; q < s; ++q) tl[(size_t)t * s + q] = pool[m.uniform_index(d.npts)];
      }
    }
    const size_t b = draw_base_h[wl];
    if (d.draws) {
      NB_CUDA(cudaMemcpyAsync(rheads.p + b, hd.data(), hd.size() * 4, cudaMemcpyHostToDevice, S));
      NB_CUDA(cudaMemcpyAsync(rtails.p + b * s, tl.data(), tl.size() * 4, cudaMemcpyHostToDevice, S));
    }
    NB_CUDA(cudaMemcpyAsync(mt_b.p + wl, &m.s, sizeof(MtState), cudaMemcpyHostToDevice, S));
    NB_CUDA(cudaStreamSynchronize(S));
  }

  // One replay epoch on the device: streams -> draws -> dependencies ->
  // dataflow SGD -> per-worker losses in draw order.
  void launch_replay_epoch(SgdParams& P) {
    cudaStream_t S = st();
    if (!df_blocks)
      df_blocks = dataflow_resident_blocks(smem_replay, ctx->sm_count, (uint32_t)k, (uint32_t)s);
    ReplayDev R = replay_dev();
    NB_CUDA(cudaMemsetAsync(reject.p, 0, reject.bytes(), S));
    NB_CUDA(cudaMemsetAsync(redges.p, 0, redges.bytes(), S));
    if (pre_ok && pre_epoch == epochs_done) {
      // this epoch's words and end state were formed during the last epoch
      std::swap(words, words2);
      std::swap(mt_b, mt_c);
      R.words = words.p;
      R.st_out = mt_b.p;
      NB_CUDA(cudaStreamWaitEvent(S, pre_ev, 0));
    } else if (nwl) {
      launch_mt_words(R, wcount.p, S);
      launched("k_mt_words");
    }
    pre_ok = false;
    if (nwl) {
      launch_replay_map(R, P, pool_d.p, pool_off_d.p, S);
      launched("k_replay_map");
    }
    std::vector<uint32_t> rj(std::max<uint32_t>(nwl, 1), 0);
    NB_CUDA(cudaMemcpyAsync(rj.data(), reject.p, rj.size() * 4, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    // (NOMAD_B200_REPLAY_HOST_DRAWS=1 takes the rejection path for every
    // worker: a test hook for the fallback, whose result must not change)
    const bool force = std::getenv("NOMAD_B200_REPLAY_HOST_DRAWS") != nullptr;
    for (uint32_t wl = 0; wl < nwl; ++wl)
      if (rj[wl] || force) host_draws(wl);
    // the next epoch's MT words on the side stream (its start state, mt_b, is
    // final now), overlapping this epoch's dependency pass
    const bool pf = prefetch && nwl && epochs_done + 1 < cfg.epochs;
    if (pf) {
      if (!side) {
        NB_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        NB_CUDA(cudaEventCreateWithFlags(&pre_ev, cudaEventDisableTiming));
        NB_CUDA(cudaEventCreateWithFlags(&map_ev, cudaEventDisableTiming));
      }
      if (!words2.p) words2.alloc(words.n);
      if (!mt_c.p) mt_c.alloc(mt_b.n);
      ReplayDev Rn = R;
      Rn.st_in = mt_b.p;
      Rn.st_out = mt_c.p;
      Rn.words = words2.p;
      NB_CUDA(cudaEventRecord(map_ev, S));  // this epoch's map read its words
      NB_CUDA(cudaStreamWaitEvent(side, map_ev, 0));
      launch_mt_words(Rn, wcount.p, side);
      launched("k_mt_words");
      NB_CUDA(cudaEventRecord(pre_ev, side));
      pre_ok = true;
      pre_epoch = epochs_done + 1;
    }
    launch_replay_deps(R, P, sort_tmp.p, sort_bytes, S);
    launched("k_replay_deps");
    // the cooperative dataflow kernel needs every SM: the side stream's work first
    if (pf) NB_CUDA(cudaStreamWaitEvent(S, pre_ev, 0));
    if (!df_blocks)
      df_blocks = dataflow_resident_blocks(smem_replay, ctx->sm_count, (uint32_t)k, (uint32_t)s);
    NB_CUDA(cudaMemsetAsync(rdone.p, 0, rdone.bytes(), S));
    NB_CUDA(cudaMemsetAsync(ticket.p, 0, 4, S));
    P.loss_slot = loss_slot.p;
    P.wk_draw_base = wk_draw_base.p;
    NB_CUDA(cudaEventRecord(ev[0], S));
    if (nwl && total_draws) {
      launch_sgd_dataflow(P, R, df_blocks, smem_replay, S);
      launched("k_sgd_dataflow");
      if (!R.followers) {  // (warp form: the dataflow kernel's followers summed them)
        launch_loss_seq(loss_slot.p, wk_draw_base.p, wk_d.p, nwl, wloss.p, S);
        launched("k_loss_seq");
      }
    }
    NB_CUDA(cudaEventRecord(ev[1], S));
    std::swap(mt_a, mt_b);  // this epoch's end state starts the next
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
    for (uint32_t a = 0; a < nwl; a += wave) {
      const uint32_t b = std::min<uint32_t>(nwl, a + wave);
      uint32_t maxc = 0;
      for (uint32_t wl = a; wl < b; ++wl) maxc = std::max(maxc, nchunk[wl]);
      for (uint32_t lc = 0; lc < maxc; ++lc)
        for (uint32_t wl = a; wl < b; ++wl)
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
  // progress (cfg.hogwild_double_float); outside a run they are f64 again.
  bool pos_is_df = false;
  void pos_format(bool df) {
    if (df == pos_is_df || !cfg.hogwild_double_float) return;
    launch_pos_df(pos.p, (uint32_t)orig_of.size(), df, st());
    launched("k_pos_df");
    pos_is_df = df;
  }

  // ------------------------------------------------ means exchange (K9)
  // This rank's cluster means into its slot (optimizer.hpp:414-433).
  void compute_means() {
    cudaStream_t S = st();
    const uint32_t ncl = (uint32_t)lcl.size();
    if (!ncl) return;
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
  // One process per rank: the all-gather of the slots over NCCL.
  void exchange_self() {
    if (world > 1 && !grouped)
      NB_NCCL(ncclAllGather(slot.p, recv.p, 2 * (size_t)max_slots, ncclDouble, comm, st()));
  }
  // The all-gathered slots -> the C-entry means snapshot (+ global cell tables).
  void unpack_means() {
    cudaStream_t S = st();
    launch_means_unpack(world > 1 ? recv.p : slot.p, slot_gid.p, (uint32_t)world * max_slots,
                        means.p, S);
    launched("k_means_unpack");
    if (gcells) {
      launch_cell_tables(means.p, wk_d.p, nwl, remote_ids.p, remote_probs.p, cell_probs.p,
                         (uint32_t)C, cfg.approx_all_but_own, (double)cfg.negatives, hog_cells,
                         gcell_mu.p, gcell_w.p, cm3.p, S);
      launched("k_cell_tables");
    }
  }
  void count_comm() {  // CommLog: one message per worker (optimizer.hpp:429-440)
    ++comm_epochs;
    comm_msgs += W;
    comm_doubles += 2 * C;
    comm_counts += C;
  }

  // ------------------------------------------------------ divergence
  // The first offender, ordered (global worker, key): replay keeps one key
  // per worker, (t * stride + u) << 32 | point, so the reported draw is the
  // first one of the lowest diverging worker — the order in which workers
  // are run one after another; throughput mode keeps one key (worker 0).
  // Point ids are mapped to original ids so every rank decodes the same way.
  DivKey host_key(const unsigned long long* keys) const {
    const uint32_t nk = cfg.sgd_mode == NOMAD_B200_SGD_REPLAY ? nwl : 1;
    for (uint32_t wl = 0; wl < nk; ++wl)
      if (keys[wl] != ~0ull)
        return DivKey{cfg.sgd_mode == NOMAD_B200_SGD_REPLAY ? (uint64_t)(w0 + wl) : 0ull,
                      (keys[wl] & 0xFFFFFFFF00000000ull) | orig_of[(uint32_t)keys[wl]]};
    return DivKey{};
  }
  DivKey local_key() {
    std::vector<unsigned long long> keys(std::max<uint32_t>(nwl, 1));
    NB_CUDA(cudaMemcpyAsync(keys.data(), diverge.p, diverge.bytes(), cudaMemcpyDeviceToHost, st()));
    NB_CUDA(cudaStreamSynchronize(st()));
    return host_key(keys.data());
  }
  // One process per rank: every rank must reach the same decision, or the
  // next collective hangs — lexicographic min over ranks (two ncclMin).
  DivKey agree_key(DivKey k) {
    if (grouped || world == 1) return k;
    DBuf<unsigned long long> kb(1);
    auto allmin = [&](uint64_t v) {
      unsigned long long x = v;
      NB_CUDA(cudaMemcpyAsync(kb.p, &x, 8, cudaMemcpyHostToDevice, st()));
      NB_NCCL(ncclAllReduce(kb.p, kb.p, 1, ncclUint64, ncclMin, comm, st()));
      NB_CUDA(cudaMemcpyAsync(&x, kb.p, 8, cudaMemcpyDeviceToHost, st()));
      NB_CUDA(cudaStreamSynchronize(st()));
      return (uint64_t)x;
    };
    const uint64_t w = allmin(k.worker);
    const uint64_t key = allmin(k.worker == w ? k.key : ~0ull);
    return DivKey{w, key};
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
    P.gcells = gcells ? 1 : 0;
    P.gcell_mu = gcell_mu.p;
    P.gcell_w = gcell_w.p;
    P.cm3 = cm3.p;
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

  double step_of(uint64_t e) const {  // optimizer.hpp:85-91, :390-391
    const double lr = lr0 * (1.0 - static_cast<double>(e) / static_cast<double>(cfg.epochs));
    return lr / static_cast<double>(cfg.batch_size);
  }

  // Continue the schedule at epoch `e` (resume from a checkpoint layout).
  // Throughput mode: draws are keyed by (seed, epoch, worker, t), nothing to
  // replay. Replay mode: each worker's mt19937_64 stream is advanced past the
  // skipped epochs' draws exactly as an epoch consumes them.
  void seek(uint64_t e) {
    if (e > cfg.epochs) fail(kParameter, "epoch out of range for schedule");
    if (cfg.sgd_mode == NOMAD_B200_SGD_REPLAY && e != epochs_done) {
      if (e < epochs_done) fail(kParameter, "replay mode cannot seek backwards");
      std::vector<Mt64> m(std::max<uint32_t>(nwl, 1));
      for (uint32_t wl = 0; wl < nwl; ++wl)
        NB_CUDA(cudaMemcpy(&m[wl].s, mt_a.p + wl, sizeof(MtState), cudaMemcpyDeviceToHost));
      for (; epochs_done < e; ++epochs_done)
        for (uint32_t wl = 0; wl < nwl; ++wl) {
          const WorkerDev& d = wk[wl];
          for (uint32_t t = 0; t < d.draws; ++t) {
            const uint32_t h = elig_h[d.elig_off + m[wl].uniform_index(d.n_elig)];
            const uint64_t pn = cfg.approx_all_but_own ? lcl[local_cluster_of(h)].count : d.npts;
            for (uint64_t q = 0; q < s; ++q) (void)m[wl].uniform_index(pn);
          }
        }
      for (uint32_t wl = 0; wl < nwl; ++wl)
        NB_CUDA(cudaMemcpy(mt_a.p + wl, &m[wl].s, sizeof(MtState), cudaMemcpyHostToDevice));
      pre_ok = false;  // a prefetched epoch is no longer the next one
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

  // ------------------------------------------- throughput run (async)
  // Every epoch's SGD kernel, means pass and exchange are queued back to
  // back; per-epoch loss / edge sums land in device arrays read once at the
  // end; divergence keys carry the run-relative epoch.
  uint64_t a_E = 0, a_first = 0;
  DBuf<double> a_loss;
  DBuf<unsigned long long> a_edge;
  std::vector<cudaEvent_t> a_ev;
  std::vector<double> a_lh, a_all;  // per epoch x local worker; multi-process: all ranks
  std::vector<unsigned long long> a_eh;
  std::vector<unsigned long long> a_keys;

  void async_begin(uint64_t E) {
    if (epochs_done + E > cfg.epochs) fail(kParameter, "epoch out of range for schedule");
    const uint64_t L = std::max<uint32_t>(nwl, 1);
    a_E = E;
    a_first = epochs_done;
    a_loss.alloc(std::max<uint64_t>(E * L, 1));
    a_edge.alloc(std::max<uint64_t>(E * L, 1));
    NB_CUDA(cudaMemsetAsync(a_loss.p, 0, a_loss.bytes(), st()));
    NB_CUDA(cudaMemsetAsync(a_edge.p, 0, a_edge.bytes(), st()));
    for (auto& x : a_ev) cudaEventDestroy(x);
    a_ev.assign(3 * E, nullptr);
    for (auto& x : a_ev) NB_CUDA(cudaEventCreate(&x));
    pos_format(true);
  }
  void async_launch(uint64_t it) {
    cudaStream_t S = st();
    const uint64_t L = std::max<uint32_t>(nwl, 1);
    SgdParams P = params(step_of(epochs_done), epochs_done);
    P.loss_acc = a_loss.p + it * L;
    P.edge_acc = a_edge.p + it * L;
    NB_CUDA(cudaMemsetAsync(chunk_counter.p, 0, 4, S));
    NB_CUDA(cudaEventRecord(a_ev[3 * it], S));
    if (hog_blocks) {
      launch_sgd_hogwild(P, hog_blocks, smem_hog, S);
      launched("k_sgd_hogwild");
    }
    NB_CUDA(cudaEventRecord(a_ev[3 * it + 1], S));
    div_tag = it;
    compute_means();
  }
  void async_finish(uint64_t it) {
    unpack_means();
    NB_CUDA(cudaEventRecord(a_ev[3 * it + 2], st()));
    count_comm();
    ++epochs_done;
  }
  void async_end() {  // results to host (collective in multi-process mode)
    cudaStream_t S = st();
    const uint64_t E = a_E, L = std::max<uint32_t>(nwl, 1);
    div_tag = 0;
    pos_format(false);
    a_lh.assign(E * L, 0.0);
    a_eh.assign(E * L, 0);
    if (E) {
      NB_CUDA(cudaMemcpyAsync(a_lh.data(), a_loss.p, E * L * 8, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaMemcpyAsync(a_eh.data(), a_edge.p, E * L * 8, cudaMemcpyDeviceToHost, S));
    }
    a_all.clear();
    if (world > 1 && !grouped && E) {
      DBuf<double> g((size_t)world * E * L);
      NB_NCCL(ncclAllGather(a_loss.p, g.p, E * L, ncclDouble, comm, S));
      a_all.resize((size_t)world * E * L);
      NB_CUDA(cudaMemcpyAsync(a_all.data(), g.p, a_all.size() * 8, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
    }
    a_keys.assign(std::max<uint32_t>(nwl, 1), ~0ull);
    NB_CUDA(cudaMemcpyAsync(a_keys.data(), diverge.p, diverge.bytes(), cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    for (uint64_t it = 0; it < E; ++it) {
      float a = 0.f, b = 0.f;
      NB_CUDA(cudaEventElapsedTime(&a, a_ev[3 * it], a_ev[3 * it + 1]));
      NB_CUDA(cudaEventElapsedTime(&b, a_ev[3 * it + 1], a_ev[3 * it + 2]));
      sgd_ms += a;
      means_ms += b;
      ++timed_epochs;
    }
    for (auto& x : a_ev) cudaEventDestroy(x);
    a_ev.clear();
    for (uint64_t i = 0; i < E * L && i < a_eh.size(); ++i)
      if (i % L < nwl) edge_updates += a_eh[i];
  }

  // -------------------------------------- replay / verbose run (per epoch sync)
  uint64_t s_E = 0;
  std::vector<double> s_wl_loss, s_all_loss;
  std::vector<unsigned long long> s_wl_edges;
  DBuf<double> s_gl;  // gathered per-worker losses (multi-process)
  uint64_t s_edges = 0;
  std::chrono::steady_clock::time_point s_t0;

  void sync_begin(uint64_t E) {
    s_E = E;
    s_wl_loss.assign(nwl, 0.0);
    s_wl_edges.assign(nwl, 0);
    s_all_loss.assign((size_t)world * std::max<uint32_t>(nwl, 1), 0.0);
    if (!ev[0])
      for (auto& x : ev) NB_CUDA(cudaEventCreate(&x));
  }
  void sync_launch(uint64_t it) {
    cudaStream_t S = st();
    const uint64_t e = epochs_done;
    if (e >= cfg.epochs) fail(kParameter, "epoch out of range for schedule");
    s_t0 = std::chrono::steady_clock::now();
    SgdParams P = params(step_of(e), e);
    s_edges = 0;
    const bool replay = cfg.sgd_mode == NOMAD_B200_SGD_REPLAY;
    if (replay) {
      launch_replay_epoch(P);
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
    compute_means();
  }
  void sync_finish() {  // after the exchange; results to host (collective in multi-process mode)
    cudaStream_t S = st();
    unpack_means();
    pos_format(false);
    NB_CUDA(cudaEventRecord(ev[2], S));
    // per-worker loss sums -> epoch mean (optimizer.hpp:444-451)
    const double* lsrc = cfg.sgd_mode == NOMAD_B200_SGD_REPLAY ? wloss.p : loss_acc.p;
    if (nwl) NB_CUDA(cudaMemcpyAsync(s_wl_loss.data(), lsrc, nwl * 8, cudaMemcpyDeviceToHost, S));
    if (nwl)
      NB_CUDA(cudaMemcpyAsync(s_wl_edges.data(),
                              cfg.sgd_mode == NOMAD_B200_SGD_HOGWILD ? edge_acc.p : redges.p,
                              nwl * 8, cudaMemcpyDeviceToHost, S));
    if (world > 1 && !grouped) {
      if (!s_gl.p) s_gl.alloc((size_t)world * nwl);
      NB_NCCL(ncclAllGather(lsrc, s_gl.p, nwl, ncclDouble, comm, S));
      NB_CUDA(cudaMemcpyAsync(s_all_loss.data(), s_gl.p, (size_t)world * nwl * 8,
                              cudaMemcpyDeviceToHost, S));
    }
  }
  DivKey sync_collect() {  // waits for this rank's epoch; returns its divergence key
    const DivKey key = local_key();  // syncs the stream
    if (cfg.sgd_mode == NOMAD_B200_SGD_REPLAY) {
      uint32_t stalled = 0;
      NB_CUDA(cudaMemcpy(&stalled, stall.p, 4, cudaMemcpyDeviceToHost));
      if (stalled) {
        // leave the mailboxes empty for any later epoch (a stalled epoch
        // may have left values in them)
        if (rmbox.p) NB_CUDA(cudaMemsetAsync(rmbox.p, 0xFF, rmbox.bytes(), st()));
        if (rlink.p) NB_CUDA(cudaMemsetAsync(loss_slot.p, 0xFF, loss_slot.bytes(), st()));
        fail(kInternal, "replay dataflow stalled (schedule watchdog)");
      }
    }
    float a = 0.f, b = 0.f;
    NB_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
    NB_CUDA(cudaEventElapsedTime(&b, ev[1], ev[2]));
    sgd_ms += a;
    means_ms += b;
    ++timed_epochs;
    for (uint32_t wl = 0; wl < nwl; ++wl) s_edges += s_wl_edges[wl];
    edge_updates += s_edges;
    return key;
  }

  uint64_t local_heads() const {
    uint64_t h = 0;
    for (auto& d : wk) h += d.draws;
    return h;
  }
  uint64_t global_heads = 0;
  // Heads of all ranks (multi-process: every rank knows the plan but only
  // its own eligibility; gathered once).
  uint64_t total_heads_global() {
    if (!global_heads) {
      DBuf<double> a(1), b((size_t)world);
      double mine = (double)local_heads();
      NB_CUDA(cudaMemcpy(a.p, &mine, 8, cudaMemcpyHostToDevice));
      NB_NCCL(ncclAllGather(a.p, b.p, 1, ncclDouble, comm, st()));
      std::vector<double> h(world);
      NB_CUDA(cudaMemcpyAsync(h.data(), b.p, world * 8, cudaMemcpyDeviceToHost, st()));
      NB_CUDA(cudaStreamSynchronize(st()));
      for (double v : h) global_heads += (uint64_t)v;
    }
    return global_heads;
  }

  // ----------------------------------------------------- layout in / out
  DBuf<double2> stage;  // n rows, original order (host <-> device staging)

  // Replace this rank's positions from a layout in ORIGINAL order (the
  // caller re-gathers the means).
  void set_rows(const double* in, int loc) {
    cudaStream_t S = st();
    const uint32_t n_loc = (uint32_t)orig_of.size();
    const double* src = in;
    if (loc != NOMAD_B200_DEVICE) {
      if (stage.n != n) stage.alloc(n);
      copy_h2d(ctx, stage.p, in, n * 16);
      src = reinterpret_cast<const double*>(stage.p);
    }
    if (n_loc) {
      launch_gather_layout(reinterpret_cast<const double2*>(src), orig_of_d.p, n_loc, pos.p, S);
      launched("k_gather_layout");
    }
  }

  // This rank's rows into `out` (ORIGINAL order); only_mine: other rows untouched.
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
    if (n_loc == n) {  // every row is local: scatter on the device, one D2H copy
      if (stage.n != n) stage.alloc(n);
      if (n_loc) {
        launch_scatter_layout(pos.p, orig_of_d.p, n_loc, stage.p, S);
        launched("k_scatter_layout");
      }
      copy_d2h(ctx, out, stage.p, n * 16);
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

}  // namespace nb

// The trainer of the C-ABI: one rank (one process per GPU) or every rank of
// a group (one process, G contexts), driven epoch by epoch in lockstep.
struct nomad_b200_trainer {
  std::vector<std::unique_ptr<RankTrainer>> r;
  nomad_b200_group* grp = nullptr;

  RankTrainer& R0() { return *r[0]; }
  bool replay() const { return r[0]->cfg.sgd_mode == NOMAD_B200_SGD_REPLAY; }
  bool multiproc() const { return !grp && r[0]->world > 1; }

  // The per-epoch all-gather of every rank's slot into every rank's recv.
  void exchange() {
    if (!grp) {
      R0().exchange_self();
      return;
    }
    if (r.size() == 1) return;
    const size_t cnt = 2 * (size_t)R0().max_slots;
    if (grp->loopback) {  // one device, one stream: device copies in program order
      for (auto& q : r)
        for (size_t src = 0; src < r.size(); ++src)
          NB_CUDA(cudaMemcpyAsync(q->recv.p + src * cnt, r[src]->slot.p, cnt * 8,
                                  cudaMemcpyDeviceToDevice, q->st()));
      return;
    }
    NB_NCCL(ncclGroupStart());
    for (auto& t : r) {
      t->bind();
      NB_NCCL(ncclAllGather(t->slot.p, t->recv.p, cnt, ncclDouble, t->comm, t->st()));
    }
    NB_NCCL(ncclGroupEnd());
  }

  void means_all() {
    for (auto& t : r) { t->bind(); t->compute_means(); }
    exchange();
    for (auto& t : r) { t->bind(); t->unpack_means(); }
  }

  // Same decision on every rank; throws Divergence (optimizer.hpp:222-225).
  void check_key(DivKey dk, uint64_t epoch_base, bool replay_key) {
    if (multiproc()) dk = R0().agree_key(dk);
    if (dk.none()) return;
    const uint64_t gk = dk.key;
    char m[200];
    const uint32_t p = (uint32_t)gk;
    if (replay_key) {
      const uint64_t stride = 2 + R0().k + R0().s;
      snprintf(m, sizeof m, "positions diverged at epoch %llu, head draw %llu (point %u)",
               (unsigned long long)epoch_base, (unsigned long long)((gk >> 32) / stride), p);
    } else {
      snprintf(m, sizeof m, "positions diverged at epoch %llu (point %u)",
               (unsigned long long)(epoch_base + (gk >> 32)), p);
    }
    fail(kDivergence, m);
  }

  void after_setup() {
    means_all();  // epoch-0 means of the init layout (optimizer.hpp:384)
    DivKey dk;
    for (auto& t : r) { t->bind(); dk = std::min(dk, t->local_key()); }
    check_key(dk, 0, false);
  }

  uint64_t all_heads() {
    if (multiproc()) return R0().total_heads_global();
    uint64_t h = 0;
    for (auto& t : r) h += t->local_heads();
    return h;
  }
  void run(uint64_t E, double* epoch_loss) {
    if (!replay() && !R0().cfg.verbose) return run_async(E, epoch_loss);
    run_sync(E, epoch_loss);
  }

  void run_async(uint64_t E, double* epoch_loss) {
    for (auto& t : r) { t->bind(); t->async_begin(E); }
    for (uint64_t it = 0; it < E; ++it) {
      for (auto& t : r) { t->bind(); t->async_launch(it); }
      exchange();
      for (auto& t : r) { t->bind(); t->async_finish(it); }
    }
    for (auto& t : r) { t->bind(); t->async_end(); }
    DivKey dk;
    for (auto& t : r) dk = std::min(dk, t->host_key(t->a_keys.data()));
    check_key(dk, R0().a_first, false);
    const uint64_t heads = all_heads();
    const size_t L = std::max<uint32_t>(R0().nwl, 1), nwl = R0().nwl;
    for (uint64_t it = 0; it < E; ++it) {
      double acc = 0.0;  // worker order: rank-major, then local worker
      if (multiproc()) {
        for (int rk = 0; rk < R0().world; ++rk)
          for (size_t wl = 0; wl < nwl; ++wl) acc += R0().a_all[((size_t)rk * E + it) * L + wl];
      } else {
        for (auto& t : r)
          for (size_t wl = 0; wl < nwl; ++wl) acc += t->a_lh[it * L + wl];
      }
      if (epoch_loss) epoch_loss[it] = heads > 0 ? acc / static_cast<double>(heads) : 0.0;
    }
  }

  void run_sync(uint64_t E, double* epoch_loss) {
    for (auto& t : r) { t->bind(); t->sync_begin(E); }
    for (uint64_t it = 0; it < E; ++it) {
      const uint64_t e = R0().epochs_done;
      for (auto& t : r) { t->bind(); t->sync_launch(it); }
      exchange();
      for (auto& t : r) { t->bind(); t->sync_finish(); }
      DivKey dk;
      for (auto& t : r) { t->bind(); dk = std::min(dk, t->sync_collect()); }
      check_key(dk, e, replay());
      double acc = 0.0;
      if (multiproc()) {
        for (double v : R0().s_all_loss) acc += v;
      } else {
        for (auto& t : r)
          for (double v : t->s_wl_loss) acc += v;
      }
      const uint64_t heads = all_heads();
      const double mean_loss = heads > 0 ? acc / static_cast<double>(heads) : 0.0;
      if (epoch_loss) epoch_loss[it] = mean_loss;
      for (auto& t : r) {
        t->count_comm();
        ++t->epochs_done;
      }
      if (R0().cfg.verbose) {
        const double secs =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - R0().s_t0).count();
        const double lr = R0().lr0 * (1.0 - static_cast<double>(e) /
                                                static_cast<double>(R0().cfg.epochs));
        std::fprintf(stderr, "epoch %llu/%llu lr %.6g loss %.6f time %.2fs\n",
                     (unsigned long long)(e + 1), (unsigned long long)R0().cfg.epochs, lr,
                     mean_loss, secs);
      }
    }
  }

  void set_layout(const double* in, int loc) {
    std::vector<double> host;
    if (loc == NOMAD_B200_DEVICE && grp && !grp->loopback && r.size() > 1) {
      R0().bind();  // ranks on other devices read a host copy
      host.resize(2 * R0().n);
      NB_CUDA(cudaMemcpy(host.data(), in, host.size() * 8, cudaMemcpyDeviceToHost));
      in = host.data();
      loc = NOMAD_B200_HOST;
    }
    for (auto& t : r) { t->bind(); t->set_rows(in, loc); }
    means_all();
    for (auto& t : r) { t->bind(); NB_CUDA(cudaStreamSynchronize(t->st())); }
  }

  void layout(double* out, int loc) {
    if (loc == NOMAD_B200_DEVICE && grp && !grp->loopback && r.size() > 1)
      fail(kParameter, "device layout output of a multi-device group: use a host buffer");
    for (auto& t : r) { t->bind(); t->layout(out, loc); }
  }
};

namespace {

// Host copies of device-resident trainer inputs (ranks on other devices).
struct HostInputs {
  std::vector<uint32_t> off, nbr, asg;
  std::vector<double> init;
  nomad_b200_graph g{};
  nomad_b200_clusters c{};
};

void to_host(const nomad_b200_graph* g, const nomad_b200_clusters* c, const double* init,
             int init_loc, HostInputs& H) {
  const uint64_t n = c->rows;
  H.g = *g;
  H.c = *c;
  if (g->location == NOMAD_B200_DEVICE) {
    H.off.resize(n + 1);
    NB_CUDA(cudaMemcpy(H.off.data(), g->offsets, (n + 1) * 4, cudaMemcpyDeviceToHost));
    H.nbr.resize(std::max<uint32_t>(H.off[n], 1));
    if (H.off[n])
      NB_CUDA(cudaMemcpy(H.nbr.data(), g->neighbors, (size_t)H.off[n] * 4, cudaMemcpyDeviceToHost));
    H.g.offsets = H.off.data();
    H.g.neighbors = H.nbr.data();
    H.g.distances = nullptr;
    H.g.location = NOMAD_B200_HOST;
  }
  if (c->location == NOMAD_B200_DEVICE) {
    H.asg.resize(n);
    NB_CUDA(cudaMemcpy(H.asg.data(), c->assignment, n * 4, cudaMemcpyDeviceToHost));
    H.c.assignment = H.asg.data();
    H.c.centroids = nullptr;
    H.c.sizes = nullptr;
    H.c.location = NOMAD_B200_HOST;
  }
  if (init_loc == NOMAD_B200_DEVICE) {
    H.init.resize(2 * n);
    NB_CUDA(cudaMemcpy(H.init.data(), init, n * 16, cudaMemcpyDeviceToHost));
  }
}

}  // namespace

extern "C" {

int32_t nomad_b200_trainer_create(nomad_b200_ctx* ctx, const nomad_b200_graph* graph,
                                  const nomad_b200_clusters* clusters, const double* init,
                                  int32_t init_loc, const nomad_b200_train_config* cfg,
                                  int32_t rank, int32_t world, const void* nccl_id,
                                  nomad_b200_trainer** out) {
  return guard([&] {
    if (!ctx || !graph || !clusters || !init || !cfg || !out) fail(kParameter, "NULL argument");
    bind_device(ctx);
    auto tr = std::make_unique<nomad_b200_trainer>();
    auto t = std::make_unique<RankTrainer>();
    t->ctx = ctx;
    t->cfg = *cfg;
    t->rank = rank;
    t->world = world;
    t->setup(graph, clusters, init, init_loc, nccl_id);
    tr->r.push_back(std::move(t));
    tr->after_setup();
    *out = tr.release();
  });
}

int32_t nomad_b200_group_trainer_create(nomad_b200_group* grp, const nomad_b200_graph* graph,
                                        const nomad_b200_clusters* clusters, const double* init,
                                        int32_t init_loc, const nomad_b200_train_config* cfg,
                                        nomad_b200_trainer** out) {
  return guard([&] {
    if (!grp || !graph || !clusters || !init || !cfg || !out) fail(kParameter, "NULL argument");
    const int G = (int)grp->ctx.size();
    auto tr = std::make_unique<nomad_b200_trainer>();
    tr->grp = grp;
    HostInputs H;
    const nomad_b200_graph* g = graph;
    const nomad_b200_clusters* c = clusters;
    const double* in = init;
    int in_loc = init_loc;
    const bool on_dev = graph->location == NOMAD_B200_DEVICE ||
                        clusters->location == NOMAD_B200_DEVICE || init_loc == NOMAD_B200_DEVICE;
    if (G > 1 && !grp->loopback && on_dev) {  // inputs live on rank 0's device
      bind_device(grp->ctx[0]);
      to_host(graph, clusters, init, init_loc, H);
      g = &H.g;
      c = &H.c;
      if (init_loc == NOMAD_B200_DEVICE) {
        in = H.init.data();
        in_loc = NOMAD_B200_HOST;
      }
    }
    for (int rk = 0; rk < G; ++rk) {
      auto t = std::make_unique<RankTrainer>();
      t->ctx = grp->ctx[rk];
      t->cfg = *cfg;
      t->rank = rk;
      t->world = G;
      t->grouped = true;
      t->prefetch = !grp->loopback;  // ranks on one device: no concurrent side-stream work
      t->comm = grp->comm.empty() ? nullptr : static_cast<ncclComm_t>(grp->comm[rk]);
      t->bind();
      t->setup(g, c, in, in_loc, nullptr);
      tr->r.push_back(std::move(t));
    }
    tr->after_setup();
    *out = tr.release();
  });
}

int32_t nomad_b200_trainer_destroy(nomad_b200_trainer* t) {
  return guard([&] {
    if (!t) return;
    for (auto& x : t->r) {
      bind_device(x->ctx);
      cudaStreamSynchronize(x->ctx->stream);
    }
    for (auto& x : t->r) {  // each rank's buffers on its own device
      bind_device(x->ctx);
      x.reset();
    }
    cudaGetLastError();  // teardown errors are not reported to later launches
    delete t;
  });
}

int32_t nomad_b200_trainer_ranks(nomad_b200_trainer* t, int32_t* ranks) {
  return guard([&] {
    if (!t || !ranks) fail(kParameter, "NULL argument");
    *ranks = (int32_t)t->r.size();
  });
}

int32_t nomad_b200_trainer_run(nomad_b200_trainer* t, uint64_t n_epochs, double* epoch_loss) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    t->run(n_epochs, epoch_loss);
  });
}

int32_t nomad_b200_trainer_layout(nomad_b200_trainer* t, double* out, int32_t loc) {
  return guard([&] {
    if (!t || !out) fail(kParameter, "NULL argument");
    t->layout(out, loc);
  });
}

int32_t nomad_b200_trainer_means(nomad_b200_trainer* t, double* means, uint32_t* counts) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    RankTrainer& R = t->R0();
    R.bind();
    if (means) {
      NB_CUDA(cudaMemcpyAsync(means, R.means.p, R.C * 16, cudaMemcpyDeviceToHost, R.st()));
      NB_CUDA(cudaStreamSynchronize(R.st()));
    }
    if (counts) std::memcpy(counts, R.sizes.data(), R.C * 4);
  });
}

int32_t nomad_b200_trainer_comm(nomad_b200_trainer* t, uint64_t* epochs, uint64_t* messages,
                                uint64_t* doubles, uint64_t* counts) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    RankTrainer& R = t->R0();
    if (epochs) *epochs = R.comm_epochs;
    if (messages) *messages = R.comm_msgs;
    if (doubles) *doubles = R.comm_doubles;
    if (counts) *counts = R.comm_counts;
  });
}

int32_t nomad_b200_trainer_set_layout(nomad_b200_trainer* t, const double* layout, int32_t loc) {
  return guard([&] {
    if (!t || !layout) fail(kParameter, "NULL argument");
    t->set_layout(layout, loc);
  });
}

int32_t nomad_b200_trainer_timing(nomad_b200_trainer* t, double* sgd_ms, double* means_ms,
                                  uint64_t* epochs) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    // device time of the slowest rank (ranks of a loopback group share one
    // GPU and run one after another: their sum)
    double a = 0.0, b = 0.0;
    for (auto& x : t->r) {
      if (t->grp && t->grp->loopback) {
        a += x->sgd_ms;
        b += x->means_ms;
      } else {
        a = std::max(a, x->sgd_ms);
        b = std::max(b, x->means_ms);
      }
    }
    if (sgd_ms) *sgd_ms = a;
    if (means_ms) *means_ms = b;
    if (epochs) *epochs = t->R0().timed_epochs;
  });
}

int32_t nomad_b200_trainer_seek(nomad_b200_trainer* t, uint64_t epoch) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    for (auto& x : t->r) x->seek(epoch);
  });
}

int32_t nomad_b200_trainer_progress(nomad_b200_trainer* t, uint64_t* epochs_done,
                                    uint64_t* edge_updates) {
  return guard([&] {
    if (!t) fail(kParameter, "trainer is NULL");
    uint64_t e = 0;
    for (auto& x : t->r) e += x->edge_updates;
    if (epochs_done) *epochs_done = t->R0().epochs_done;
    if (edge_updates) *edge_updates = e;
  });
}

}  // extern "C"
