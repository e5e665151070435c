// SGD epoch kernels and cluster-means kernels (see sgd_kernels.cuh).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "sgd_device.cuh"
#include "sgd_kernels.cuh"

namespace nb {

// ------------------------------------------------------- K8r replay kernel
//
// P.replay_ctas CTAs per local worker (a cooperative launch, so all are
// resident). The host turned the worker's mt19937_64 draw stream into a tape
// and grouped draws into wavefront levels: draws of one level touch
// pairwise-disjoint points, and every draw comes after all earlier draws (in
// sequential order t) that touch any of its points. So executing level by
// level — the worker's CTAs split a level's draws, then meet at a per-worker
// barrier in global memory — performs exactly the reference's sequential
// per-worker update sequence (optimizer.hpp:253-304). Positions are read
// through L2 (ld.global.cg), so a CTA sees the previous level's updates made
// on other SMs. Each draw runs the reference arithmetic in its op order with
// _rn intrinsics (no FMA), so positions are bit-identical.
__device__ __forceinline__ double2 ldpos(const double2* p) { return __ldcg(p); }

__global__ void __launch_bounds__(256) k_sgd_replay(SgdParams P) {
  extern __shared__ __align__(16) double sm[];
  const uint32_t K = P.replay_ctas ? P.replay_ctas : 1;
  const uint32_t w = blockIdx.x / K, part = blockIdx.x % K;
  const WorkerDev W = P.workers[w];
  const uint32_t k = P.k, s = P.s, C = P.n_clusters;
  // shared tables: weights (k+1)*k, then means/probs of all C cells (or,
  // when 3C doubles do not fit, the same [C][3] table in global memory)
  double* wt = sm;
  double* cms = sm + (k + 1) * k;  // 3*C: mu.x, mu.y, p
  for (uint32_t i = threadIdx.x; i < (k + 1) * k; i += blockDim.x) wt[i] = P.wtab[i];
  if (!P.gcells)
    for (uint32_t r = threadIdx.x; r < C; r += blockDim.x) {
      cms[3 * r] = P.means[r].x;
      cms[3 * r + 1] = P.means[r].y;
      cms[3 * r + 2] = P.cell_probs[r];
    }
  const double* cm = P.gcells ? P.cm3 : cms;
  __syncthreads();
  const double M = (double)P.m_total;
  const uint32_t lvl0 = P.wk_lvl_base[w], nlev = P.wk_nlev[w];
  const uint32_t stride = 2 + k + s;
  for (uint32_t L = 0; L < nlev; ++L) {
    const uint32_t b = P.lvl_off[lvl0 + L], e = P.lvl_off[lvl0 + L + 1];
    for (uint32_t i = b + part * blockDim.x + threadIdx.x; i < e; i += K * blockDim.x) {
      const uint32_t head = P.tape_head[i];
      const uint32_t* tails = P.tape_tails + (size_t)i * s;
      const uint32_t t = P.tape_t[i];
      const double2 h = ldpos(P.pos + head);
      // noise terms (objective.hpp:113-145)
      uint32_t own = 0;
      double lm = W.local_mass;
      if (P.all_but_own) {
        own = P.lclusters[P.cl_of[head]].gid;
        lm = P.cell_probs[own];
      }
      double remote_sum = 0.0;
      const uint32_t nr = P.all_but_own ? C : W.n_rem;
      for (uint32_t q = 0; q < nr; ++q) {
        const uint32_t r = P.all_but_own ? q : P.remote_ids[W.rem_off + q];
        if (P.all_but_own && r == own) continue;
        const double qr = cauchy_rn(h.x, h.y, cm[3 * r], cm[3 * r + 1]);
        remote_sum = __dadd_rn(remote_sum, __dmul_rn(cm[3 * r + 2], qr));
      }
      const double mean_field = __dmul_rn(M, remote_sum);
      const double sf = __ddiv_rn(__dmul_rn(M, lm), (double)s);
      double qsum = 0.0;
      for (uint32_t q = 0; q < s; ++q) {
        const double2 o = ldpos(P.pos + tails[q]);
        qsum = __dadd_rn(qsum, cauchy_rn(h.x, h.y, o.x, o.y));
      }
      const double bg = __dadd_rn(mean_field, __dmul_rn(sf, qsum));
      // attraction (objective.hpp:197-213)
      const uint32_t cnt = P.ncnt ? P.ncnt[head] : k;
      const uint32_t* nb = P.ell + (size_t)head * P.kpad;
      const double* wrow = wt + cnt * k;
      double loss = 0.0, bgs = 0.0, gx = 0.0, gy = 0.0;
      double gn[2 * 64];
      for (uint32_t j = 0; j < cnt; ++j) {
        const double2 o = ldpos(P.pos + nb[j]);
        const double q = cauchy_rn(h.x, h.y, o.x, o.y);
        const double wj = wrow[j];
        const double qb = __dadd_rn(q, bg);
        loss = __dadd_rn(loss, __dmul_rn(wj, -log(__ddiv_rn(q, qb))));
        bgs = __dadd_rn(bgs, __ddiv_rn(wj, qb));
        const double pull = __dmul_rn(
            __dmul_rn(__dmul_rn(__dmul_rn(2.0, wj),
                                __dsub_rn(__ddiv_rn(1.0, q), __ddiv_rn(1.0, qb))),
                      q),
            q);
        const double dx = __dsub_rn(h.x, o.x), dy = __dsub_rn(h.y, o.y);
        gx = __dadd_rn(gx, __dmul_rn(pull, dx));
        gy = __dadd_rn(gy, __dmul_rn(pull, dy));
        gn[2 * j] = __dmul_rn(-pull, dx);
        gn[2 * j + 1] = __dmul_rn(-pull, dy);
      }
      // negative repulsion (objective.hpp:216-226)
      double gm[2 * 16];
      for (uint32_t q = 0; q < s; ++q) {
        const double2 o = ldpos(P.pos + tails[q]);
        const double qn = cauchy_rn(h.x, h.y, o.x, o.y);
        const double push = __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, bgs), sf), qn), qn);
        const double dx = __dsub_rn(h.x, o.x), dy = __dsub_rn(h.y, o.y);
        gx = __dsub_rn(gx, __dmul_rn(push, dx));
        gy = __dsub_rn(gy, __dmul_rn(push, dy));
        gm[2 * q] = __dmul_rn(push, dx);
        gm[2 * q + 1] = __dmul_rn(push, dy);
      }
      // mean repulsion (objective.hpp:229-236)
      for (uint32_t q = 0; q < nr; ++q) {
        const uint32_t r = P.all_but_own ? q : P.remote_ids[W.rem_off + q];
        if (P.all_but_own && r == own) continue;
        const double mx = cm[3 * r], my = cm[3 * r + 1];
        const double qr = cauchy_rn(h.x, h.y, mx, my);
        const double push = __dmul_rn(
            __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, bgs), M), cm[3 * r + 2]), qr), qr);
        gx = __dsub_rn(gx, __dmul_rn(push, __dsub_rn(h.x, mx)));
        gy = __dsub_rn(gy, __dmul_rn(push, __dsub_rn(h.y, my)));
      }
      P.loss_slot[P.wk_draw_base[w] + t] = loss;
      // apply (optimizer.hpp:215-227, :293-303): head, neighbours, tails
      const double st = P.step;
      uint32_t u = 0;
      auto apply = [&](uint32_t p, double ax, double ay) {
        double2 v = ldpos(P.pos + p);
        v.x = __dsub_rn(v.x, __dmul_rn(st, ax));
        v.y = __dsub_rn(v.y, __dmul_rn(st, ay));
        P.pos[p] = v;
        if (diverged(v.x, v.y))
          atomicMin(P.diverge + w, ((unsigned long long)t * stride + u) << 32 | p);
        ++u;
      };
      apply(head, gx, gy);
      if (!P.head_only) {
        for (uint32_t j = 0; j < cnt; ++j) apply(nb[j], gn[2 * j], gn[2 * j + 1]);
        for (uint32_t q = 0; q < s; ++q) apply(tails[q], gm[2 * q], gm[2 * q + 1]);
      }
    }
    // level barrier across the worker's CTAs
    __syncthreads();
    if (K > 1) {
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(P.replay_bar + w, 1u);
        const uint32_t target = (L + 1) * K;
        while (*reinterpret_cast<volatile uint32_t*>(P.replay_bar + w) < target) {
        }
        __threadfence();
      }
      __syncthreads();
    }
  }
}

// Per-worker loss in sequential draw order (optimizer.hpp:289-290).
__global__ void k_loss_seq(const double* slot, const uint32_t* base, const WorkerDev* wk,
                           uint32_t nw, double* out) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nw) return;
  double acc = 0.0;
  const double* p = slot + base[w];
  for (uint32_t t = 0; t < wk[w].draws; ++t) acc = __dadd_rn(acc, p[t]);
  out[w] = acc;
}

// ------------------------------------------------------ K9 cluster means
//
// Exact: per local cluster and coordinate, a sequential sum over the
// cluster's contiguous segment (ascending original id == the order of
// gather_means, optimizer.hpp:163-168 / :420-428), then / count.
__global__ void k_means_exact(const double2* pos, const LocalCluster* lc, uint32_t ncl,
                              double* slot /* ncl x 2 */) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= 2 * ncl) return;
  const uint32_t c = g >> 1, dim = g & 1;
  const LocalCluster L = lc[c];
  const double* p = reinterpret_cast<const double*>(pos) + 2 * (size_t)L.start + dim;
  double acc = 0.0;
  for (uint32_t i = 0; i < L.count; ++i) acc = __dadd_rn(acc, p[2 * (size_t)i]);
  slot[g] = __ddiv_rn(acc, (double)L.count);
}

// Throughput: chunked tree reduction into per-cluster sums (atomics), fused
// with the divergence scan of every position (optimizer.hpp:220-221).
// DF: positions are double-float rows {hi.x, hi.y, lo.x, lo.y} (the
// throughput kernel's atomic format); each row is read as hi + lo and
// renormalised in place (hi = fl32(p), lo = fl32(p - hi)).
template <bool DF>
__global__ void k_means_chunk(double2* pos, const LocalCluster* lc, uint32_t ncl,
                              uint32_t chunk, const uint32_t* chunk_off, double* sums,
                              unsigned long long* diverge, unsigned long long tag) {
  __shared__ double red[8];
  // find cluster for this block
  uint32_t c = 0;
  while (c + 1 < ncl && blockIdx.x >= chunk_off[c + 1]) ++c;
  const LocalCluster L = lc[c];
  const uint32_t b0 = L.start + (blockIdx.x - chunk_off[c]) * chunk;
  const uint32_t b1 = min(b0 + chunk, L.start + L.count);
  double sx = 0.0, sy = 0.0;
  for (uint32_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    double2 v;
    if constexpr (DF) {
      float4* r = reinterpret_cast<float4*>(pos) + i;
      const float4 f = *r;
      v = make_double2((double)f.x + (double)f.z, (double)f.y + (double)f.w);
      const float hx = __double2float_rn(v.x), hy = __double2float_rn(v.y);
      *r = make_float4(hx, hy, __double2float_rn(v.x - (double)hx), __double2float_rn(v.y - (double)hy));
    } else {
      v = pos[i];
    }
    if (diverged(v.x, v.y)) atomicMin(diverge, (tag << 32) | (unsigned long long)i);
    sx += v.x;
    sy += v.y;
  }
  sx = block_sum(sx, red);
  sy = block_sum(sy, red);
  if (threadIdx.x == 0) {
    atomicAdd(&sums[2 * c], sx);
    atomicAdd(&sums[2 * c + 1], sy);
  }
}

// In-place format change of the position rows: f64 (x, y) <-> double-float.
__global__ void k_pos_df(double2* pos, uint32_t n, int to_df) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (to_df) {
    const double2 v = pos[i];
    const float hx = __double2float_rn(v.x), hy = __double2float_rn(v.y);
    reinterpret_cast<float4*>(pos)[i] =
        make_float4(hx, hy, __double2float_rn(v.x - (double)hx), __double2float_rn(v.y - (double)hy));
  } else {
    const float4 f = reinterpret_cast<const float4*>(pos)[i];
    pos[i] = make_double2((double)f.x + (double)f.z, (double)f.y + (double)f.w);
  }
}

__global__ void k_means_finalize(double* sums, const LocalCluster* lc, uint32_t ncl,
                                 double* slot) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= 2 * ncl) return;
  slot[g] = sums[g] / (double)lc[g >> 1].count;
  sums[g] = 0.0;
}

// Scatter gathered slots into the C-entry means table (static map).
__global__ void k_means_unpack(const double* recv, const uint32_t* slot_gid, uint32_t nslots,
                               double2* means) {
  const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nslots) return;
  const uint32_t gid = slot_gid[g];
  if (gid != 0xFFFFFFFFu) means[gid] = make_double2(recv[2 * g], recv[2 * g + 1]);
}

// Local ELL graph in local ids from the global CSR in original ids. A list
// longer than k, or a neighbour that is not a point of the row's own worker
// shard (another rank's, or another worker's on this rank), is rejected:
// positive edges stay inside a shard (optimizer.hpp:292-300).
__global__ void k_build_ell(const uint32_t* offsets, const uint32_t* nbrs,
                            const uint32_t* orig_of, const uint32_t* new_of,
                            const uint32_t* cl_of, const LocalCluster* lcl, uint32_t n_loc,
                            uint32_t k, uint32_t kpad, uint32_t* ell, uint8_t* ncnt,
                            unsigned long long* bad) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_loc) return;
  const uint32_t o = orig_of[i];
  const uint32_t b = offsets[o], c = offsets[o + 1] - b;
  if (c > k) { atomicMin(bad, (unsigned long long)i); return; }
  const uint32_t wi = lcl[cl_of[i]].worker;
  for (uint32_t t = 0; t < kpad; ++t) {
    uint32_t v = i;  // pad with self (never read beyond count)
    if (t < c) {
      v = new_of[nbrs[b + t]];
      if (v == 0xFFFFFFFFu || lcl[cl_of[v]].worker != wi) {
        atomicMin(bad, (unsigned long long)i);
        v = i;
      }
    }
    ell[(size_t)i * kpad + t] = v;
  }
  if (ncnt) ncnt[i] = (uint8_t)c;
}

// Global-memory cell tables (see launch_cell_tables).
__global__ void k_cell_tables(const double2* means, const WorkerDev* wk, uint32_t nwl,
                              const uint32_t* remote_ids, const double* remote_probs,
                              const double* cell_probs, uint32_t C, int abo, double M,
                              uint32_t stride, double2* gmu, double* gw, double* cm3) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.y == nwl) {  // replay table
    if (q < C) {
      cm3[3 * (size_t)q] = means[q].x;
      cm3[3 * (size_t)q + 1] = means[q].y;
      cm3[3 * (size_t)q + 2] = cell_probs[q];
    }
    return;
  }
  const WorkerDev W = wk[blockIdx.y];
  const uint32_t ncell = abo ? C : W.n_rem;
  if (q >= ncell) return;
  const uint32_t r = abo ? q : remote_ids[W.rem_off + q];
  const double p = abo ? cell_probs[r] : remote_probs[W.rem_off + q];
  gmu[(size_t)blockIdx.y * stride + q] = means[r];
  gw[(size_t)blockIdx.y * stride + q] = M * p;
}

// Layout in original order: out[orig_of[i]] = pos[i].
__global__ void k_scatter_layout(const double2* pos, const uint32_t* orig_of, uint32_t n_loc,
                                 double2* out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_loc) out[orig_of[i]] = pos[i];
}
__global__ void k_gather_layout(const double2* in, const uint32_t* orig_of, uint32_t n_loc,
                                double2* pos) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_loc) pos[i] = in[orig_of[i]];
}

// ------------------------------------------------------ host launchers

static unsigned blocks_for(uint64_t n, unsigned t) { return (unsigned)((n + t - 1) / t); }

uint32_t replay_ctas_per_worker(uint32_t n_workers, size_t smem, int sm_count) {
  if (smem > 48 * 1024)
    NB_CUDA(cudaFuncSetAttribute(k_sgd_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  NB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sgd_replay, 256, smem));
  const uint32_t resident = (uint32_t)std::max(per_sm, 1) * (uint32_t)sm_count;
  return std::max<uint32_t>(1, std::min<uint32_t>(32, resident / std::max<uint32_t>(n_workers, 1)));
}

void launch_sgd_replay(const SgdParams& P, uint32_t n_workers, size_t smem, cudaStream_t st) {
  if (smem > 48 * 1024)
    NB_CUDA(cudaFuncSetAttribute(k_sgd_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (P.replay_ctas > 1) {
    NB_CUDA(cudaMemsetAsync(P.replay_bar, 0, n_workers * sizeof(uint32_t), st));
    SgdParams Pc = P;
    void* args[] = {&Pc};
    NB_CUDA(cudaLaunchCooperativeKernel((const void*)k_sgd_replay, dim3(n_workers * P.replay_ctas),
                                        dim3(256), args, smem, st));
  } else {
    k_sgd_replay<<<n_workers, 256, smem, st>>>(P);
  }
}

void launch_loss_seq(const double* slot, const uint32_t* base, const WorkerDev* wk, uint32_t nw,
                     double* out, cudaStream_t st) {
  k_loss_seq<<<blocks_for(nw, 32), 32, 0, st>>>(slot, base, wk, nw, out);
}

void launch_means_exact(const double2* pos, const LocalCluster* lc, uint32_t ncl, double* slot,
                        cudaStream_t st) {
  k_means_exact<<<blocks_for(2 * ncl, 64), 64, 0, st>>>(pos, lc, ncl, slot);
}

void launch_means_chunk(double2* pos, bool df, const LocalCluster* lc, uint32_t ncl, uint32_t chunk,
                        const uint32_t* chunk_off, uint32_t nchunks, double* sums,
                        unsigned long long* diverge, unsigned long long tag, cudaStream_t st) {
  if (df)
    k_means_chunk<true><<<nchunks, 256, 0, st>>>(pos, lc, ncl, chunk, chunk_off, sums, diverge, tag);
  else
    k_means_chunk<false><<<nchunks, 256, 0, st>>>(pos, lc, ncl, chunk, chunk_off, sums, diverge, tag);
}

void launch_pos_df(double2* pos, uint32_t n, bool to_df, cudaStream_t st) {
  if (n) k_pos_df<<<blocks_for(n, 256), 256, 0, st>>>(pos, n, to_df ? 1 : 0);
}

void launch_means_finalize(double* sums, const LocalCluster* lc, uint32_t ncl, double* slot,
                           cudaStream_t st) {
  k_means_finalize<<<blocks_for(2 * ncl, 64), 64, 0, st>>>(sums, lc, ncl, slot);
}

void launch_means_unpack(const double* recv, const uint32_t* slot_gid, uint32_t nslots,
                         double2* means, cudaStream_t st) {
  k_means_unpack<<<blocks_for(nslots, 128), 128, 0, st>>>(recv, slot_gid, nslots, means);
}

void launch_build_ell(const uint32_t* offsets, const uint32_t* nbrs, const uint32_t* orig_of,
                      const uint32_t* new_of, const uint32_t* cl_of, const LocalCluster* lcl,
                      uint32_t n_loc, uint32_t k, uint32_t kpad, uint32_t* ell, uint8_t* ncnt,
                      unsigned long long* bad, cudaStream_t st) {
  k_build_ell<<<blocks_for(n_loc, 256), 256, 0, st>>>(offsets, nbrs, orig_of, new_of, cl_of, lcl,
                                                      n_loc, k, kpad, ell, ncnt, bad);
}

void launch_cell_tables(const double2* means, const WorkerDev* wk, uint32_t nwl,
                        const uint32_t* remote_ids, const double* remote_probs,
                        const double* cell_probs, uint32_t C, int all_but_own, double M,
                        uint32_t stride, double2* gmu, double* gw, double* cm3, cudaStream_t st) {
  const dim3 grid(blocks_for(std::max<uint32_t>(std::max(stride, C), 1), 128), nwl + 1);
  k_cell_tables<<<grid, 128, 0, st>>>(means, wk, nwl, remote_ids, remote_probs, cell_probs, C,
                                      all_but_own, M, stride, gmu, gw, cm3);
}

void launch_scatter_layout(const double2* pos, const uint32_t* orig_of, uint32_t n_loc,
                           double2* out, cudaStream_t st) {
  k_scatter_layout<<<blocks_for(n_loc, 256), 256, 0, st>>>(pos, orig_of, n_loc, out);
}

void launch_gather_layout(const double2* in, const uint32_t* orig_of, uint32_t n_loc,
                          double2* pos, cudaStream_t st) {
  k_gather_layout<<<blocks_for(n_loc, 256), 256, 0, st>>>(in, orig_of, n_loc, pos);
}

}  // namespace nb
