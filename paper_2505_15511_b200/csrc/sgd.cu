// SGD epoch kernels and cluster-means kernels (see sgd_kernels.cuh).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "sgd_kernels.cuh"

namespace nb {

// ---------------------------------------------------------------- helpers

// Exact Cauchy kernel, reference op order, no contraction (objective.hpp:36-41).
__device__ __forceinline__ double cauchy_rn(double a0, double a1, double b0, double b1) {
  const double dx = __dsub_rn(a0, b0), dy = __dsub_rn(a1, b1);
  const double sq = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  return __ddiv_rn(1.0, __dadd_rn(1.0, sq));
}

// Fast fp64 reciprocal for throughput mode: MUFU.RCP64H seed + one cubic
// Newton correction (rel. error ~2^-69 before rounding => ~1 ulp).
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// optimizer.hpp:220-221 divergence predicate.
__device__ __forceinline__ bool diverged(double x, double y) {
  return !isfinite(x) || !isfinite(y) || fabs(x) > 1e9 || fabs(y) > 1e9;
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;  // valid on thread 0
}

// ------------------------------------------------------- K8r replay kernel
//
// One CTA per local worker. The host turned the worker's mt19937_64 draw
// stream into a tape and grouped draws into wavefront levels: draws of one
// level touch pairwise-disjoint points, and every draw comes after all
// earlier draws (in sequential order t) that touch any of its points. So
// executing level by level, with a CTA barrier between levels, performs
// exactly the reference's sequential per-worker update sequence
// (optimizer.hpp:253-304). Each draw runs the reference arithmetic in its
// op order with _rn intrinsics (no FMA), so positions are bit-identical.
__global__ void __launch_bounds__(256) k_sgd_replay(SgdParams P) {
  extern __shared__ __align__(16) double sm[];
  const uint32_t w = blockIdx.x;
  const WorkerDev W = P.workers[w];
  const uint32_t k = P.k, s = P.s, C = P.n_clusters;
  // shared tables: weights (k+1)*k, then means/probs of all C cells
  double* wt = sm;
  double* cm = sm + (k + 1) * k;  // 3*C: mu.x, mu.y, p
  for (uint32_t i = threadIdx.x; i < (k + 1) * k; i += blockDim.x) wt[i] = P.wtab[i];
  for (uint32_t r = threadIdx.x; r < C; r += blockDim.x) {
    cm[3 * r] = P.means[r].x;
    cm[3 * r + 1] = P.means[r].y;
    cm[3 * r + 2] = P.cell_probs[r];
  }
  __syncthreads();
  const double M = (double)P.m_total;
  const uint32_t lvl0 = P.wk_lvl_base[w], nlev = P.wk_nlev[w];
  const uint32_t stride = 2 + k + s;
  for (uint32_t L = 0; L < nlev; ++L) {
    const uint32_t b = P.lvl_off[lvl0 + L], e = P.lvl_off[lvl0 + L + 1];
    for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      const uint32_t head = P.tape_head[i];
      const uint32_t* tails = P.tape_tails + (size_t)i * s;
      const uint32_t t = P.tape_t[i];
      const double2 h = P.pos[head];
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
        const double2 o = P.pos[tails[q]];
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
        const double2 o = P.pos[nb[j]];
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
        const double2 o = P.pos[tails[q]];
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
        double2 v = P.pos[p];
        v.x = __dsub_rn(v.x, __dmul_rn(st, ax));
        v.y = __dsub_rn(v.y, __dmul_rn(st, ay));
        P.pos[p] = v;
        if (diverged(v.x, v.y))
          atomicMin(P.diverge, ((unsigned long long)t * stride + u) << 32 | p);
        ++u;
      };
      apply(head, gx, gy);
      if (!P.head_only) {
        for (uint32_t j = 0; j < cnt; ++j) apply(nb[j], gn[2 * j], gn[2 * j + 1]);
        for (uint32_t q = 0; q < s; ++q) apply(tails[q], gm[2 * q], gm[2 * q + 1]);
      }
    }
    __syncthreads();
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

// ------------------------------------------------------ K8p hogwild kernel
//
// Throughput mode, thread per head. Draws come from Philox4x32-10 keyed by
// (seed, epoch, worker, draw t): head ~ U(eligible_w), tails ~ U(pool_w)
// exactly as optimizer.hpp:254-255/:284-285 define the distributions. All
// (1 + k + s) rows are gathered up front (MLP), the gradient is the
// reference's (objective.hpp:178-237) with algebraic reuse
// (pull = 2 w q bg / (q + bg), mean push folded into one sum), and updates
// are fp64 atomic scatter-adds (RED.ADD.F64). Heads in flight per worker are
// bounded by the grid share the host gives the worker (hogwild cap).
template <int KMAX, int SMAX>
__global__ void __launch_bounds__(256, 2) k_sgd_hogwild(SgdParams P) {
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[8];
  uint32_t w = 0;
  while (w + 1 < P.n_workers && blockIdx.x >= P.workers[w + 1].blk_start) ++w;
  const WorkerDev W = P.workers[w];
  const uint32_t k = P.k, s = P.s, C = P.n_clusters;
  const double M = (double)P.m_total;
  double* wt = sm;                              // (k+1)*k
  double* tab = sm + (((k + 1) * k + 1) & ~1u);  // 3 per cell: mu.x, mu.y, M*p
  const uint32_t ncell = P.all_but_own ? C : W.n_rem;
  for (uint32_t i = threadIdx.x; i < (k + 1) * k; i += blockDim.x) wt[i] = P.wtab[i];
  for (uint32_t q = threadIdx.x; q < ncell; q += blockDim.x) {
    const uint32_t r = P.all_but_own ? q : P.remote_ids[W.rem_off + q];
    const double p = P.all_but_own ? P.cell_probs[r] : P.remote_probs[W.rem_off + q];
    tab[3 * q] = P.means[r].x;
    tab[3 * q + 1] = P.means[r].y;
    tab[3 * q + 2] = M * p;
  }
  __syncthreads();

  const uint32_t nthr = W.nblk * blockDim.x;
  const uint32_t tid = (blockIdx.x - W.blk_start) * blockDim.x + threadIdx.x;
  const double sf_w = M * W.local_mass / (double)s;
  const double st = P.step;
  double loss_acc = 0.0;
  unsigned long long edges = 0;
  for (uint32_t t = tid; t < W.draws; t += nthr) {
    // --- draws (1 + s) x 64 bits
    uint64_t rnd[2 * ((SMAX + 2) / 2)];
#pragma unroll
    for (int c = 0; c < (SMAX + 2) / 2; ++c) {
      const u32x4 r = philox4x32_10(u32x4{t, W.id, (uint32_t)P.epoch, (uint32_t)c},
                                    P.seed_lo, P.seed_hi);
      rnd[2 * c] = join64(r.x, r.y);
      rnd[2 * c + 1] = join64(r.z, r.w);
    }
    const uint32_t head = P.elig[W.elig_off + bounded(rnd[0], W.n_elig)];
    uint32_t pool0 = W.pstart, pooln = W.npts, own_gid = 0xFFFFFFFFu;
    double sf = sf_w;
    if (P.all_but_own) {
      const LocalCluster L = P.lclusters[P.cl_of[head]];
      pool0 = L.start;
      pooln = L.count;
      own_gid = L.gid;
      sf = M * P.cell_probs[L.gid] / (double)s;
    }
    // --- gathers
    const uint32_t cnt = P.ncnt ? P.ncnt[head] : k;
    uint32_t nb[KMAX];
    const uint32_t* row = P.ell + (size_t)head * P.kpad;
#pragma unroll
    for (int j = 0; j < KMAX; j += 4) {
      const uint4 v = *reinterpret_cast<const uint4*>(row + j);
      nb[j] = v.x; nb[j + 1] = v.y; nb[j + 2] = v.z; nb[j + 3] = v.w;
    }
    uint32_t tl[SMAX];
#pragma unroll
    for (int q = 0; q < SMAX; ++q) tl[q] = q < (int)s ? pool0 + bounded(rnd[1 + q], pooln) : 0;
    const double2 h = P.pos[head];
    double2 pn[KMAX], pt[SMAX];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) pn[j] = j < (int)cnt ? P.pos[nb[j]] : make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < SMAX; ++q) pt[q] = q < (int)s ? P.pos[tl[q]] : make_double2(0.0, 0.0);

    // --- mean field: S1 = M sum p q, S2 = M sum p q^2 (h - mu)
    double s1 = 0.0, s2x = 0.0, s2y = 0.0;
    for (uint32_t q = 0; q < ncell; ++q) {
      if (P.all_but_own && q == own_gid) continue;
      const double dx = h.x - tab[3 * q], dy = h.y - tab[3 * q + 1];
      const double qq = frcp(fma(dx, dx, fma(dy, dy, 1.0)));
      const double pq = tab[3 * q + 2] * qq;
      s1 += pq;
      const double pq2 = pq * qq;
      s2x = fma(pq2, dx, s2x);
      s2y = fma(pq2, dy, s2y);
    }
    // --- sampled negatives
    double qn[SMAX], qsum = 0.0;
#pragma unroll
    for (int q = 0; q < SMAX; ++q) {
      if (q < (int)s) {
        const double dx = h.x - pt[q].x, dy = h.y - pt[q].y;
        qn[q] = frcp(fma(dx, dx, fma(dy, dy, 1.0)));
        qsum += qn[q];
      }
    }
    const double bg = fma(sf, qsum, s1);
    // --- attraction; neighbour updates issued immediately
    const double* wrow = wt + cnt * k;
    double gx = 0.0, gy = 0.0, bgs = 0.0;
    float lf = 0.f;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
      if (j < (int)cnt) {
        const double dx = h.x - pn[j].x, dy = h.y - pn[j].y;
        const double q = frcp(fma(dx, dx, fma(dy, dy, 1.0)));
        const double inv = frcp(q + bg);
        const double wj = wrow[j];
        lf -= (float)wj * __logf((float)(q * inv));
        bgs = fma(wj, inv, bgs);
        const double pull = 2.0 * wj * q * bg * inv;
        gx = fma(pull, dx, gx);
        gy = fma(pull, dy, gy);
        if (!P.head_only) {
          const double a = st * pull;
          atomicAdd(&P.pos[nb[j]].x, a * dx);
          atomicAdd(&P.pos[nb[j]].y, a * dy);
        }
      }
    }
    // --- negative repulsion
    const double c2 = 2.0 * bgs * sf;
#pragma unroll
    for (int q = 0; q < SMAX; ++q) {
      if (q < (int)s) {
        const double dx = h.x - pt[q].x, dy = h.y - pt[q].y;
        const double push = c2 * qn[q] * qn[q];
        gx = fma(-push, dx, gx);
        gy = fma(-push, dy, gy);
        if (!P.head_only) {
          const double a = -st * push;
          atomicAdd(&P.pos[tl[q]].x, a * dx);
          atomicAdd(&P.pos[tl[q]].y, a * dy);
        }
      }
    }
    // --- mean repulsion, then the head update
    gx = fma(-2.0 * bgs, s2x, gx);
    gy = fma(-2.0 * bgs, s2y, gy);
    atomicAdd(&P.pos[head].x, -st * gx);
    atomicAdd(&P.pos[head].y, -st * gy);
    loss_acc += (double)lf;
    edges += cnt + s;
  }
  const double ls = block_sum(loss_acc, red);
  const double es = block_sum((double)edges, red);
  if (threadIdx.x == 0) {
    atomicAdd(&P.loss_acc[w], ls);
    atomicAdd(&P.edge_acc[w], (unsigned long long)es);
  }
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
__global__ void k_means_chunk(const double2* pos, const LocalCluster* lc, uint32_t ncl,
                              uint32_t chunk, const uint32_t* chunk_off, double* sums,
                              unsigned long long* diverge) {
  __shared__ double red[8];
  // find cluster for this block
  uint32_t c = 0;
  while (c + 1 < ncl && blockIdx.x >= chunk_off[c + 1]) ++c;
  const LocalCluster L = lc[c];
  const uint32_t b0 = L.start + (blockIdx.x - chunk_off[c]) * chunk;
  const uint32_t b1 = min(b0 + chunk, L.start + L.count);
  double sx = 0.0, sy = 0.0;
  for (uint32_t i = b0 + threadIdx.x; i < b1; i += blockDim.x) {
    const double2 v = pos[i];
    if (diverged(v.x, v.y)) atomicMin(diverge, (unsigned long long)i);
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

// Local ELL graph in local ids from the global CSR in original ids.
__global__ void k_build_ell(const uint32_t* offsets, const uint32_t* nbrs,
                            const uint32_t* orig_of, const uint32_t* new_of, uint32_t n_loc,
                            uint32_t kpad, uint32_t* ell, uint8_t* ncnt,
                            unsigned long long* bad) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_loc) return;
  const uint32_t o = orig_of[i];
  const uint32_t b = offsets[o], c = offsets[o + 1] - b;
  if (c > kpad) { atomicMin(bad, (unsigned long long)i); return; }
  for (uint32_t t = 0; t < kpad; ++t) {
    uint32_t v = i;  // pad with self (never read beyond count)
    if (t < c) {
      v = new_of[nbrs[b + t]];
      if (v == 0xFFFFFFFFu) { atomicMin(bad, (unsigned long long)i); v = i; }
    }
    ell[(size_t)i * kpad + t] = v;
  }
  if (ncnt) ncnt[i] = (uint8_t)c;
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

void launch_sgd_replay(const SgdParams& P, uint32_t n_workers, size_t smem, cudaStream_t st) {
  if (smem > 48 * 1024)
    NB_CUDA(cudaFuncSetAttribute(k_sgd_replay, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_sgd_replay<<<n_workers, 256, smem, st>>>(P);
}

void launch_loss_seq(const double* slot, const uint32_t* base, const WorkerDev* wk, uint32_t nw,
                     double* out, cudaStream_t st) {
  k_loss_seq<<<blocks_for(nw, 32), 32, 0, st>>>(slot, base, wk, nw, out);
}

void launch_sgd_hogwild(const SgdParams& P, uint32_t nblocks, size_t smem, cudaStream_t st) {
  if (P.s > 8) fail(kParameter, "throughput mode supports local_draws <= 8");
  auto go = [&](auto kern) {
    if (smem > 48 * 1024)
      NB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<nblocks, 256, smem, st>>>(P);
  };
  if (P.kpad <= 16 && P.s == 5) go(k_sgd_hogwild<16, 5>);
  else if (P.kpad <= 16) go(k_sgd_hogwild<16, 8>);
  else if (P.kpad <= 32) go(k_sgd_hogwild<32, 8>);
  else if (P.kpad <= 64) go(k_sgd_hogwild<64, 8>);
  else fail(kParameter, "throughput mode supports k <= 64");
}

uint32_t hogwild_resident_blocks(uint32_t kpad, uint32_t s, size_t smem, int sm_count) {
  int per_sm = 0;
  auto q = [&](auto kern) {
    if (smem > 48 * 1024)
      NB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    NB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
  };
  if (kpad <= 16 && s == 5) q(k_sgd_hogwild<16, 5>);
  else if (kpad <= 16) q(k_sgd_hogwild<16, 8>);
  else if (kpad <= 32) q(k_sgd_hogwild<32, 8>);
  else q(k_sgd_hogwild<64, 8>);
  return (uint32_t)std::max(1, per_sm) * (uint32_t)sm_count;
}

void launch_means_exact(const double2* pos, const LocalCluster* lc, uint32_t ncl, double* slot,
                        cudaStream_t st) {
  k_means_exact<<<blocks_for(2 * ncl, 64), 64, 0, st>>>(pos, lc, ncl, slot);
}

void launch_means_chunk(const double2* pos, const LocalCluster* lc, uint32_t ncl, uint32_t chunk,
                        const uint32_t* chunk_off, uint32_t nchunks, double* sums,
                        unsigned long long* diverge, cudaStream_t st) {
  k_means_chunk<<<nchunks, 256, 0, st>>>(pos, lc, ncl, chunk, chunk_off, sums, diverge);
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
                      const uint32_t* new_of, uint32_t n_loc, uint32_t kpad, uint32_t* ell,
                      uint8_t* ncnt, unsigned long long* bad, cudaStream_t st) {
  k_build_ell<<<blocks_for(n_loc, 256), 256, 0, st>>>(offsets, nbrs, orig_of, new_of, n_loc,
                                                      kpad, ell, ncnt, bad);
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
