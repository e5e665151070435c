// K8p: throughput-mode SGD epoch kernel (optimizer.hpp:232-307 semantics with
// Hogwild-style concurrent heads).
//
// One group of G lanes per head (G = 4: 8 heads per warp). Draws come from
// Philox4x32-10 keyed by (seed, epoch, worker, draw t): head ~ U(eligible_w),
// tails ~ U(pool_w) — the distributions of optimizer.hpp:254-255 / :284-285.
// Lane gl of a group owns neighbours [NPL*gl, NPL*gl+NPL) (one vector load of
// the ELL row), tails gl, gl+G, ..., and remote cells gl, gl+G, ...; the
// shared sums (mean field, sampled noise, bg sensitivity, head gradient) are
// butterfly-reduced inside the group, which leaves bitwise-identical values
// on every lane. The gradient is the reference's (objective.hpp:178-237)
// with algebraic reuse: pull = 2 w q bg / (q + bg), and the mean push folded
// into one sum; all arithmetic in fp64. Updates are atomic scatter-adds onto
// double-float position rows (one RED.F32x2 per row, see ld_row/add_row).
//
// Scheduling: blocks pull fixed-size chunks of draws from a global counter;
// the chunk map orders them in waves of shards (round-robin inside a wave),
// so at any moment the GPU works on a few shards whose positions stay
// resident in L2. Shards are
// disjoint and the means snapshot is read-only, so the order in which shards
// run does not change the semantics (the reference runs them as independent
// threads). Heads in flight <= grid threads / G (the hogwild cap).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "sgd_device.cuh"
#include "sgd_kernels.cuh"

// Tuning knobs (compile-time; the Makefile default is the measured best).
#ifndef HOG_MINB
#define HOG_MINB 3        // min resident blocks per SM (register cap)
#endif
#ifndef HOG_G16
#define HOG_G16 4         // lanes per head when k <= 16
#endif
// a head needs (s + 2) / 2 Philox blocks, one per lane of its group: s <= 7 needs 4 lanes
static_assert(HOG_G16 >= 4, "HOG_G16 < 4 cannot draw s = 7 negatives per head");
#ifndef HOG_ROUNDS
#define HOG_ROUNDS 8      // rounds of 256/G heads per scheduled chunk
#endif

namespace nb {

template <int G>
__device__ __forceinline__ double gsum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Position rows. DF (double-float): 16-byte rows {hi.x, hi.y, lo.x, lo.y},
// value = hi + lo (exact in fp64), updates are one RED.F32x2 onto lo (the
// per-request cost of RED.F32x2 equals one RED.F64, tools/micro/red_bench.cu,
// so a row update costs half); the means pass renormalises every epoch.
// Otherwise f64 rows and two RED.F64 per row update.
template <bool DF>
__device__ __forceinline__ double2 ld_row(const double2* pos, uint32_t i) {
  if constexpr (DF) {
    const float4 r = reinterpret_cast<const float4*>(pos)[i];
    return make_double2((double)r.x + (double)r.z, (double)r.y + (double)r.w);
  } else {
    return pos[i];
  }
}
template <bool DF>
__device__ __forceinline__ void add_row(double2* pos, uint32_t i, double ax, double ay) {
  if constexpr (DF) {
    float* lo = reinterpret_cast<float*>(pos + i) + 2;
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(lo), "f"(__double2float_rn(ax)),
                 "f"(__double2float_rn(ay))
                 : "memory");
  } else {
    atomicAdd(&pos[i].x, ax);
    atomicAdd(&pos[i].y, ay);
  }
}

// f64 rows, lane pairs: lanes 2i and 2i+1 of a group exchange one component
// of their row updates and then write x and y of the SAME row in one RED.F64
// instruction, so the two 8-byte reductions share one L1->L2 request: 2
// instructions per two rows instead of 2 per row (tools/micro/red_bench.cu:
// 196.8 G row-updates/s for lane pairs vs 98.1 G for 2x RED.F64 per lane,
// profiles/r1_red_bench.txt). Called by every lane of the warp (shuffles);
// id = 0xFFFFFFFF for no update.
__device__ __forceinline__ void pair_red(double2* pos, uint32_t id, double ux, double uy, int e) {
  const double recv = __shfl_xor_sync(0xffffffffu, e ? ux : uy, 1);
  const uint32_t pid = __shfl_xor_sync(0xffffffffu, id, 1);
  double* q = reinterpret_cast<double*>(pos);
  const uint32_t r1 = e ? pid : id;  // the even lane's row: x by the even, y by the odd lane
  if (r1 != 0xFFFFFFFFu) atomicAdd(q + 2 * (size_t)r1 + e, e ? recv : ux);
  const uint32_t r2 = e ? id : pid;  // the odd lane's row
  if (r2 != 0xFFFFFFFFu) atomicAdd(q + 2 * (size_t)r2 + e, e ? uy : recv);
}

template <int NPL>
__device__ __forceinline__ void load_ids(const uint32_t* p, uint32_t (&v)[NPL]) {
  if constexpr (NPL == 4) {
    const uint4 x = *reinterpret_cast<const uint4*>(p);
    v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
  } else if constexpr (NPL == 2) {
    const uint2 x = *reinterpret_cast<const uint2*>(p);
    v[0] = x.x; v[1] = x.y;
  } else {
#pragma unroll
    for (int j = 0; j < NPL; j += 4) {
      const uint4 x = *reinterpret_cast<const uint4*>(p + j);
      v[j] = x.x; v[j + 1] = x.y; v[j + 2] = x.z; v[j + 3] = x.w;
    }
  }
}

// One head's draws: head, tails owned by this lane, this lane's neighbour ids.
template <int NPL, int TPL>
struct Draw {
  uint32_t head, cnt, own_gid;
  uint32_t tl[TPL], nb[NPL];
  double sf;
  bool act;
};

template <int G, int KMAX, int SMAX, bool DF, bool ABO>
__global__ void __launch_bounds__(256, HOG_MINB) k_sgd_hogwild(SgdParams P) {
  constexpr int NPL = KMAX / G;            // neighbour slots per lane
  constexpr int TPL = (SMAX + G - 1) / G;  // tail slots per lane
  constexpr int GPB = 256 / G;             // heads per block per round
  extern __shared__ __align__(16) double sm[];
  __shared__ double red[8];
  __shared__ uint32_t s_chunk;
  const uint32_t k = P.k, s = P.s, C = P.n_clusters;
  const double M = (double)P.m_total;
  const int gl = threadIdx.x % G;
  const int grp = threadIdx.x / G;
  const int g0 = (threadIdx.x & 31) & ~(G - 1);  // first lane of my group
  double* wt = sm;
  // cell table: means (double2, 16-byte aligned) then weights
  double2* tmu = reinterpret_cast<double2*>(sm + ((((k + 1) * k) + 1) & ~1u));
  for (uint32_t i = threadIdx.x; i < (k + 1) * k; i += blockDim.x) wt[i] = P.wtab[i];

  double* tpw = reinterpret_cast<double*>(tmu + P.max_cells);
  uint32_t cur = 0xFFFFFFFFu;
  WorkerDev W{};
  uint32_t ncell = 0;
  double sf_w = 0.0, loss_acc = 0.0, edge_acc = 0.0;
  const double st = P.step;
  const uint32_t nblk_draw = (s + 2) / 2;  // Philox blocks per head (2 draws each)

  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_chunk = atomicAdd(P.chunk_counter, 1u);
    __syncthreads();
    const uint32_t c = s_chunk;
    uint32_t w = 0, lchunk = 0;
    if (c < P.total_chunks) {
      const uint2 cm = P.chunk_map[c];
      w = cm.x;
      lchunk = cm.y;
    }
    if (c >= P.total_chunks || w != cur) {  // block-uniform
      if (cur != 0xFFFFFFFFu) {  // flush the previous shard's statistics
        const double ls = block_sum(loss_acc, red);
        const double es = block_sum(edge_acc, red);
        if (threadIdx.x == 0) {
          atomicAdd(&P.loss_acc[cur], ls);
          atomicAdd(&P.edge_acc[cur], (unsigned long long)es);
        }
        loss_acc = 0.0;
        edge_acc = 0.0;
      }
      if (c >= P.total_chunks) break;
      cur = w;
      W = P.workers[w];
      ncell = ABO ? C : W.n_rem;
      sf_w = M * W.local_mass / (double)s;
      __syncthreads();
      if (!P.gcells)
        for (uint32_t q = threadIdx.x; q < ncell; q += blockDim.x) {
          const uint32_t r = ABO ? q : P.remote_ids[W.rem_off + q];
          const double p = ABO ? P.cell_probs[r] : P.remote_probs[W.rem_off + q];
          tmu[q] = P.means[r];  // cell means, then their weights M p_r
          tpw[q] = M * p;
        }
      __syncthreads();
    }
    const uint32_t t_base = lchunk * P.chunk_heads;
    // draw(t): the Philox draws of head t (lane b of the group computes
    // Philox block b = draws 2b, 2b+1), its tails, and the load of its
    // neighbour ids (this lane's slice of the ELL row). Executed by full warps
    // (shuffles): chunk_heads is a multiple of GPB, so every warp runs the
    // same number of rounds; inactive groups at the end of a shard run
    // predicated off.
    auto draw = [&](uint32_t t, Draw<NPL, TPL>& D) {
      D.act = t < W.draws;
      uint64_t dA = 0, dB = 0;
      if (gl < (int)nblk_draw) {
        const u32x4 r = philox4x32_10(u32x4{t, W.id, (uint32_t)P.epoch, (uint32_t)gl},
                                      P.seed_lo, P.seed_hi);
        dA = join64(r.x, r.y);
        dB = join64(r.z, r.w);
      }
      const uint64_t d0 = __shfl_sync(0xffffffffu, dA, g0);
      const uint32_t hidx = D.act ? bounded(d0, W.n_elig) : 0u;
      D.head = (W.all_elig || !D.act) ? W.pstart + hidx : P.elig[W.elig_off + hidx];
      uint32_t pool0 = W.pstart, pooln = W.npts;
      D.own_gid = 0xFFFFFFFFu;
      D.sf = sf_w;
      if constexpr (ABO) {  // optimizer.hpp:264-277
        const LocalCluster L = P.lclusters[P.cl_of[D.head]];
        pool0 = L.start;
        pooln = L.count;
        D.own_gid = L.gid;
        D.sf = M * P.cell_probs[L.gid] / (double)s;
      }
      // tails owned by this lane: q = gl + G m uses draw 1 + q
#pragma unroll
      for (int m = 0; m < TPL; ++m) {
        const int q = gl + G * m;
        const int d = 1 + q;
        const int src = g0 + (((d >> 1) < G) ? (d >> 1) : 0);
        const uint64_t a = __shfl_sync(0xffffffffu, dA, src);
        const uint64_t b = __shfl_sync(0xffffffffu, dB, src);
        D.tl[m] = (D.act && q < (int)s) ? pool0 + bounded((d & 1) ? b : a, pooln) : D.head;
      }
      D.cnt = D.act ? (P.ncnt ? P.ncnt[D.head] : k) : 0u;
      load_ids<NPL>(P.ell + (size_t)D.head * P.kpad + NPL * gl, D.nb);
    };
    Draw<NPL, TPL> D;
    draw(t_base + grp, D);
    for (uint32_t j = grp; j < P.chunk_heads; j += GPB) {
      const bool act = D.act;
      const uint32_t head = D.head, cnt = D.cnt, own_gid = D.own_gid;
      const double sf = D.sf;
      // ---- gathers (all issued before any use)
      const double2 h = ld_row<DF>(P.pos, head);
      double2 pn[NPL], pt[TPL];
#pragma unroll
      for (int i = 0; i < NPL; ++i) pn[i] = (NPL * gl + i < (int)cnt) ? ld_row<DF>(P.pos, D.nb[i]) : h;
#pragma unroll
      for (int m = 0; m < TPL; ++m) pt[m] = (act && gl + G * m < (int)s) ? ld_row<DF>(P.pos, D.tl[m]) : h;
      const bool more = j + GPB < P.chunk_heads;  // warp-uniform
      // next head's draws and neighbour ids in flight during this head's math
      Draw<NPL, TPL> Dn;
      if (more) draw(t_base + j + GPB, Dn);

      // ---- mean field over this lane's cells: S1 = M sum p q, S2 = M sum p q^2 (h - mu)
      // (own cell skipped in AllButOwn mode)
      double s1 = 0.0, s2x = 0.0, s2y = 0.0;
      {
        const uint32_t skip = ABO ? own_gid : 0xFFFFFFFFu;
        // cell table in shared memory, or (many clusters) this worker's row
        // of the global tables; inlined twice so each loop keeps its space
        auto field = [&](const double2* mu, const double* wv) {
          uint32_t q = gl;
#pragma unroll 2
          for (; q < ncell; q += G) {
            const double2 ma = mu[q];
            const double wa = q == skip ? 0.0 : wv[q];
            const double ax = h.x - ma.x, ay = h.y - ma.y;
            const double qa = frcp(fma(ax, ax, fma(ay, ay, 1.0)));
            const double pa = wa * qa;
            s1 += pa;
            const double pa2 = pa * qa;
            s2x = fma(pa2, ax, s2x);
            s2y = fma(pa2, ay, s2y);
          }
        };
        if (P.gcells)
          field(P.gcell_mu + (size_t)cur * P.max_cells, P.gcell_w + (size_t)cur * P.max_cells);
        else
          field(tmu, tpw);
      }
      // ---- sampled negatives
      double qn[TPL], qsum = 0.0;
#pragma unroll
      for (int m = 0; m < TPL; ++m) {
        qn[m] = 0.0;
        if (act && gl + G * m < (int)s) {
          const double dx = h.x - pt[m].x, dy = h.y - pt[m].y;
          qn[m] = frcp(fma(dx, dx, fma(dy, dy, 1.0)));
          qsum += qn[m];
        }
      }
      s1 = gsum<G>(s1);
      qsum = gsum<G>(qsum);
      const double bg = fma(sf, qsum, s1);
      // ---- attraction over this lane's neighbours; their updates go out now
      const double* wrow = wt + cnt * k;
      double gx = 0.0, gy = 0.0, bgs = 0.0;
      float lf = 0.f;
#pragma unroll
      for (int i = 0; i < NPL; ++i) {
        const int jj = NPL * gl + i;
        uint32_t uid = 0xFFFFFFFFu;
        double ux = 0.0, uy = 0.0;
        if (jj < (int)cnt) {
          const double dx = h.x - pn[i].x, dy = h.y - pn[i].y;
          const double q = frcp(fma(dx, dx, fma(dy, dy, 1.0)));
          const double inv = frcp(q + bg);
          const double wj = wrow[jj];
          lf -= (float)wj * __logf((float)(q * inv));
          bgs = fma(wj, inv, bgs);
          const double pull = 2.0 * wj * q * bg * inv;
          gx = fma(pull, dx, gx);
          gy = fma(pull, dy, gy);
          if (!P.head_only) {
            const double a = st * pull;
            uid = D.nb[i];
            ux = a * dx;
            uy = a * dy;
            if constexpr (DF) add_row<DF>(P.pos, uid, ux, uy);
          }
        }
        if constexpr (!DF) pair_red(P.pos, uid, ux, uy, gl & 1);
      }
      bgs = gsum<G>(bgs);
      // ---- negative repulsion
      const double c2 = 2.0 * bgs * sf;
#pragma unroll
      for (int m = 0; m < TPL; ++m) {
        uint32_t uid = 0xFFFFFFFFu;
        double ux = 0.0, uy = 0.0;
        if (act && gl + G * m < (int)s) {
          const double dx = h.x - pt[m].x, dy = h.y - pt[m].y;
          const double push = c2 * qn[m] * qn[m];
          gx = fma(-push, dx, gx);
          gy = fma(-push, dy, gy);
          if (!P.head_only) {
            const double a = -st * push;
            uid = D.tl[m];
            ux = a * dx;
            uy = a * dy;
            if constexpr (DF) add_row<DF>(P.pos, uid, ux, uy);
          }
        }
        if constexpr (!DF) pair_red(P.pos, uid, ux, uy, gl & 1);
      }
      // ---- mean repulsion + head update (lane 0 of the group)
      gx = gsum<G>(fma(-2.0 * bgs, s2x, gx));
      gy = gsum<G>(fma(-2.0 * bgs, s2y, gy));
      if constexpr (DF) {
        if (act && gl == 0) add_row<DF>(P.pos, head, -st * gx, -st * gy);
      } else {  // x by lane 0, y by lane 1 of the group: one RED.F64 instruction
        if (act && gl < 2) atomicAdd(reinterpret_cast<double*>(P.pos) + 2 * (size_t)head + gl,
                                     gl ? -st * gy : -st * gx);
      }
      if (act && gl == 0) edge_acc += (double)(cnt + s);
      loss_acc += (double)lf;
      if (more) D = Dn;
    }
  }
}

template <int G, int KMAX, int SMAX>
static void hog_go(const SgdParams& P0, uint32_t nblocks, size_t smem, cudaStream_t st,
                   int* per_sm) {
  const SgdParams& P = P0;
  // all-but-own-cluster ablation (optimizer.hpp:264-277) as a template flag: the default
  // mode keeps no per-head pool / own-cell registers
  auto kern = P.double_float
                  ? (P.all_but_own ? k_sgd_hogwild<G, KMAX, SMAX, true, true> : k_sgd_hogwild<G, KMAX, SMAX, true, false>)
                  : (P.all_but_own ? k_sgd_hogwild<G, KMAX, SMAX, false, true> : k_sgd_hogwild<G, KMAX, SMAX, false, false>);
  if (smem > 48 * 1024)
    NB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (per_sm) {
    NB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, kern, 256, smem));
    return;
  }
  kern<<<nblocks, 256, smem, st>>>(P);
}

static void hog_dispatch(const SgdParams& P, uint32_t kpad, uint32_t s, uint32_t nblocks,
                         size_t smem, cudaStream_t st, int* per_sm) {
  if (s > 15) fail(kParameter, "throughput mode supports local_draws <= 15");
  if (kpad <= 16 && s <= 7) {
    if (s <= 4) hog_go<HOG_G16, 16, 4>(P, nblocks, smem, st, per_sm);
    else hog_go<HOG_G16, 16, 8>(P, nblocks, smem, st, per_sm);
  } else if (kpad <= 16) {
    hog_go<8, 16, 16>(P, nblocks, smem, st, per_sm);
  } else if (kpad <= 32) {
    hog_go<8, 32, 16>(P, nblocks, smem, st, per_sm);
  } else if (kpad <= 64) {
    hog_go<8, 64, 16>(P, nblocks, smem, st, per_sm);
  } else {
    fail(kParameter, "throughput mode supports k <= 64");
  }
}

uint32_t hogwild_group_size(uint32_t kpad, uint32_t s) {
  return (kpad <= 16 && s <= 7) ? HOG_G16 : 8;
}
uint32_t hogwild_chunk_rounds() { return HOG_ROUNDS; }

void launch_sgd_hogwild(const SgdParams& P, uint32_t nblocks, size_t smem, cudaStream_t st) {
  hog_dispatch(P, P.kpad, P.s, nblocks, smem, st, nullptr);
}

uint32_t hogwild_resident_blocks(uint32_t kpad, uint32_t s, size_t smem, int sm_count) {
  int per_sm = 0;
  hog_dispatch(SgdParams{}, kpad, s, 0, smem, nullptr, &per_sm);
  return (uint32_t)std::max(1, per_sm) * (uint32_t)sm_count;
}

}  // namespace nb
