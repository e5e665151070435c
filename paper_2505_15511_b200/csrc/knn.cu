// K6 + K7: exact within-cluster kNN graph (knn.hpp:51-109) on the GPU.
//
// Pass 1 (filter, FFMA): per cluster, a block takes 64 query points and
// streams every 128-point candidate tile of the same cluster through shared
// memory, computing fp32 direct-difference distances sum (a - b)^2. Each
// query keeps its KP smallest approximate distances (threshold + shared
// buffer, compacted by a warp when it passes KP entries).
// Pass 2 (re-rank + certificate): a warp per query recomputes the KP
// survivors with the reference's fp64 j-ascending chain (bit-identical
// distances), sorts by (distance, id) and keeps min(k, size-1). The fp32
// chain has relative error <= g32 = (d+3)u32 against the exact distance and
// the reference's fp64 chain <= g64 = d u64, so every excluded candidate has
// reference distance >= T / (1 + g32) * (1 - g64), T = the KP-th approximate
// distance. If that bound is above the k-th re-ranked distance, the top-k is
// certified exact; otherwise the query goes to pass 3.
// Pass 3 (fallback, rare): exhaustive fp64 for uncertified queries.
#include <cub/cub.cuh>

#include <algorithm>
#include <type_traits>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "index_common.cuh"

namespace nb {

namespace {

constexpr int QT = 64;    // queries per block
constexpr int CT = 128;   // candidates per tile
constexpr int DK = 32;    // dims per smem chunk

template <int KP, int CAP = KP + CT>
__device__ void compact_warp(float* bd, uint32_t* bi, uint32_t& cnt, float& tau, int lane) {
  // keep the KP smallest (dist) of cnt <= CAP entries, by repeated
  // warp-wide min extraction; tau = KP-th smallest.
  constexpr int PER = (CAP + 31) / 32;
  float v[PER];
  uint32_t id[PER];
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    const uint32_t p = lane + 32 * e;
    v[e] = p < cnt ? bd[p] : __int_as_float(0x7f800000);
    id[e] = p < cnt ? bi[p] : 0xFFFFFFFFu;
  }
  __syncwarp();
  float last = __int_as_float(0x7f800000);
  for (int r = 0; r < KP; ++r) {
    // local min
    float m = v[0];
    int me = 0;
#pragma unroll
    for (int e = 1; e < PER; ++e)
      if (v[e] < m) { m = v[e]; me = e; }
    float wm = m;
    int wl = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, wm, o);
      const int ol = __shfl_xor_sync(0xffffffffu, wl, o);
      if (om < wm || (om == wm && ol < wl)) { wm = om; wl = ol; }
    }
    uint32_t wid = 0;
#pragma unroll
    for (int e = 0; e < PER; ++e)
      if (lane == wl && e == me) wid = id[e];
    wid = __shfl_sync(0xffffffffu, wid, wl);
    if (lane == wl) {
#pragma unroll
      for (int e = 0; e < PER; ++e)
        if (e == me) v[e] = __int_as_float(0x7f800000);
    }
    if (lane == 0) {
      bd[r] = wm;
      bi[r] = wid;
    }
    last = wm;
  }
  __syncwarp();
  if (lane == 0) {
    cnt = KP;
    tau = last;
  }
  __syncwarp();
}

// Pass 1 (FFMA filter). grid = query tiles of 64; block 256 = 16 x 16
// threads; thread (tx, ty) owns queries ty + 16 i (4) and candidates
// tx + 16 c (8) of each 128-candidate tile; distances are fp32 j-ascending
// chains sum (a - b)^2.
//  * the 32-dim chunks of the query and candidate tiles are double-buffered
//    in shared memory by cp.async (16-byte pieces when rows are
//    float4-addressable, else four 4-byte copies per piece), the next chunk
//    in flight while the current one is consumed; each thread owns six fixed
//    pieces per chunk, so the only per-tile address work is four row ids;
//  * rows are stored unpadded with the 16-byte pieces XOR-swizzled by
//    (row & 7), so the compute loop reads float4s (one LDS.128 feeds four
//    dims) without bank conflicts;
//  * queries come from their own list (the whole cluster, the rows a
//    tensor-core certificate left open, or a metric's sample); self-pairs
//    are excluded by id; members == nullptr means candidates are the rows
//    [beg, beg + size) themselves;
//  * insertions run in phases of 64 (KP = 32) or 32 (KP = 64) candidates per
//    query, so the survivor buffers hold KP + 64 / KP + 32 entries and two
//    CTAs fit per SM.
struct FilterSeg {
  uint64_t beg;    // candidates: members[beg, beg + size)
  uint64_t qbeg;   // queries: qlist[qbeg, qbeg + qn)
  uint32_t size;
  uint32_t qn;
  uint32_t qtile;  // first query tile of this segment
  uint32_t part;   // candidate partition (slot-indexed output)
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

template <int KP, bool V4>
__global__ void __launch_bounds__(256, 2) k_knn_filter(const float* __restrict__ x, uint32_t d,
                                                       const uint32_t* __restrict__ members,
                                                       const uint32_t* __restrict__ qlist,
                                                       const FilterSeg* segs, uint32_t nseg,
                                                       int by_slot /* 0: by point id; P: slot * P + part */,
                                                       uint32_t* cand_ids,
                                                       float* cand_tau, uint32_t* cand_cnt,
                                                       double lbf) {
  constexpr int NPH = KP <= 32 ? 2 : 4;    // insertion phases per tile
  constexpr int CPP = 8 / NPH;             // candidates per thread per phase
  constexpr int CAP = KP + CT / NPH;
  constexpr int ROWS = QT + CT;           // rows per chunk buffer
  constexpr int BUF = ROWS * DK;          // floats per chunk buffer
  extern __shared__ __align__(16) unsigned char smraw[];
  float* tb = reinterpret_cast<float*>(smraw);  // 2 x BUF
  float* bd = tb + 2 * BUF;
  uint32_t* bi = reinterpret_cast<uint32_t*>(bd + QT * CAP);
  uint32_t* cnt = bi + QT * CAP;
  float* tau = reinterpret_cast<float*>(cnt + QT);
  uint32_t* qid = reinterpret_cast<uint32_t*>(tau + QT);
  __shared__ int any_full;

  uint32_t s = 0;
  {
    uint32_t lo = 0, hi = nseg;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) / 2;
      if (segs[mid].qtile <= blockIdx.x) lo = mid; else hi = mid;
    }
    s = lo;
  }
  const FilterSeg S = segs[s];
  const uint32_t q0 = (blockIdx.x - S.qtile) * QT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = threadIdx.x; q < QT; q += 256) {
    cnt[q] = 0;
    tau[q] = __int_as_float(0x7f800000);
    qid[q] = q0 + q < S.qn ? qlist[S.qbeg + q0 + q] : 0xFFFFFFFFu;
  }
  // this thread's pieces: rows r_e = threadIdx.x / 8 + 32 e (e < 6; e < 2 are
  // query rows), 16-byte piece pc = threadIdx.x & 7 of each row's chunk
  const int pr = threadIdx.x >> 3, pc = threadIdx.x & 7;
  const float* qrow[2];
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const uint32_t qq = q0 + pr + 32 * e;
    qrow[e] = qq < S.qn ? x + (uint64_t)qlist[S.qbeg + qq] * d : nullptr;
  }
  const float* crow[4];
  auto load_crow = [&](uint32_t c0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t cl = c0 + pr + 32 * e;
      crow[e] = cl < S.size ? x + (members ? (uint64_t)members[S.beg + cl] : S.beg + cl) * d
                            : nullptr;
    }
  };
  const uint32_t smem_tb = (uint32_t)__cvta_generic_to_shared(tb);
  // piece (row, pc) of chunk j0 -> buffer b; swizzled slot pc ^ (row & 7)
  auto issue = [&](int b, uint32_t j0) {
    const uint32_t jb = j0 + 4 * pc;
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      const int row = pr + 32 * e;
      const float* rp = e < 2 ? qrow[e] : crow[e - 2];
      const uint32_t dst = smem_tb + (uint32_t)((b * BUF + row * DK + ((pc ^ (row & 7)) << 2)) * 4);
      if constexpr (V4) {
        const bool ok = rp != nullptr && jb < d;
        cp_async16(dst, ok ? (const void*)(rp + jb) : (const void*)x, ok ? 16u : 0u);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool ok = rp != nullptr && jb + u < d;
          cp_async4(dst + 4 * u, ok ? (const void*)(rp + jb + u) : (const void*)x, ok ? 4u : 0u);
        }
      }
    }
  };
  const uint32_t nchunk = (d + DK - 1) / DK;
  load_crow(0);
  issue(0, 0);
  cp_async_commit();
  uint32_t it = 0;  // global chunk counter (buffer = it & 1)
  for (uint32_t c0 = 0; c0 < S.size; c0 += CT) {
    float acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[i][c] = 0.f;
    for (uint32_t ch = 0; ch < nchunk; ++ch, ++it) {
      // prefetch the next chunk (next tile's first chunk at the end of a tile)
      if (ch + 1 < nchunk) {
        issue((it + 1) & 1, (ch + 1) * DK);
      } else if (c0 + CT < S.size) {
        load_crow(c0 + CT);
        issue((it + 1) & 1, 0);
      }
      cp_async_commit();
      cp_async_wait1();
      __syncthreads();
      const float* Q = tb + (it & 1) * BUF;
      const float* Cc = Q + QT * DK;
#pragma unroll
      for (int p = 0; p < DK / 4; ++p) {
        float4 qv[4], cv[8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          qv[i] = *reinterpret_cast<const float4*>(Q + (ty + 16 * i) * DK + ((p ^ (ty & 7)) << 2));
#pragma unroll
        for (int c = 0; c < 8; ++c)
          cv[c] = *reinterpret_cast<const float4*>(Cc + (tx + 16 * c) * DK + ((p ^ (tx & 7)) << 2));
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            float df = qv[i].x - cv[c].x;
            acc[i][c] = fmaf(df, df, acc[i][c]);
            df = qv[i].y - cv[c].y;
            acc[i][c] = fmaf(df, df, acc[i][c]);
            df = qv[i].z - cv[c].z;
            acc[i][c] = fmaf(df, df, acc[i][c]);
            df = qv[i].w - cv[c].w;
            acc[i][c] = fmaf(df, df, acc[i][c]);
          }
      }
      __syncthreads();
    }
    // insert below-threshold candidates, CT / NPH per query at a time
#pragma unroll
    for (int h = 0; h < NPH; ++h) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int q = ty + 16 * i;
        const uint32_t gq = qid[q];
        if (gq == 0xFFFFFFFFu) continue;
        const float t = tau[q];
#pragma unroll
        for (int c = CPP * h; c < CPP * h + CPP; ++c) {
          const uint32_t cl = c0 + tx + 16 * c;
          if (cl < S.size && acc[i][c] < t) {
            const uint32_t gid = members ? members[S.beg + cl] : (uint32_t)(S.beg + cl);
            if (gid != gq) {
              const uint32_t pos = atomicAdd(&cnt[q], 1u);
              bd[q * CAP + pos] = acc[i][c];
              bi[q * CAP + pos] = gid;
            }
          }
        }
      }
      if (threadIdx.x == 0) any_full = 0;
      __syncthreads();
      for (int q = threadIdx.x; q < QT; q += 256)
        if (cnt[q] > KP) any_full = 1;
      __syncthreads();
      if (any_full) {
        for (int q = warp; q < QT; q += 8)
          if (cnt[q] > KP) compact_warp<KP, CAP>(bd + q * CAP, bi + q * CAP, cnt[q], tau[q], lane);
        __syncthreads();
      }
    }
  }
  // survivors, indexed by point id (graph build) or by query slot (metrics)
  for (int q = warp; q < QT; q += 8) {
    const uint32_t gq = qid[q];
    if (gq == 0xFFFFFFFFu) continue;
    const uint64_t o = by_slot ? (S.qbeg + q0 + q) * (uint64_t)by_slot + S.part : gq;
    const uint32_t c = cnt[q];
    if (lane < (int)c) cand_ids[o * KP + lane] = bi[q * CAP + lane];
    if (KP > 32 && lane + 32 < (int)c) cand_ids[o * KP + lane + 32] = bi[q * CAP + lane + 32];
    if (lane == 0) {
      cand_cnt[o] = c;
      cand_tau[o] = c == KP ? __double2float_rd((double)tau[q] * lbf) : __int_as_float(0x7f800000);
    }
  }
}

// Per-label column sums over an index list (lab == nullptr: one label):
// grid (ceil(d / 128), 64 row chunks); sums[2][d], cnts[2] (atomics: the
// bisection is a heuristic, not part of any certified result).
__global__ void k_label_sums(const float* __restrict__ xr, const uint32_t* __restrict__ idx,
                             uint64_t cnt, uint32_t d, const uint8_t* __restrict__ lab,
                             double* sums, unsigned long long* cnts) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t r0 = cnt * blockIdx.y / gridDim.y, r1 = cnt * (blockIdx.y + 1) / gridDim.y;
  double a0 = 0.0, a1 = 0.0;
  unsigned long long n0 = 0, n1 = 0;
  for (uint64_t i = r0; i < r1; ++i) {
    const int l = lab ? lab[i] : 0;
    const double v = j < d ? (double)xr[(uint64_t)idx[i] * d + j] : 0.0;
    if (l) { a1 += v; ++n1; } else { a0 += v; ++n0; }
  }
  if (j < d) {
    atomicAdd(sums + j, a0);
    atomicAdd(sums + d + j, a1);
  }
  if (j == 0) {
    atomicAdd(cnts, n0);
    atomicAdd(cnts + 1, n1);
  }
}
__global__ void k_means_from_sums(const double* sums, const unsigned long long* cnts, uint32_t d,
                                  double* cen) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < 2 * d; e += gridDim.x * blockDim.x) {
    const unsigned long long c = cnts[e / d];
    cen[e] = c ? sums[e] / (double)c : 0.0;
  }
}
// one block: v = y / ||y|| (v unchanged when y == 0)
__global__ void k_normalize(const double* y, uint32_t d, double* v) {
  __shared__ double red[32];
  double a = 0.0;
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) a += y[j] * y[j];
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x < 32) {
    a = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (threadIdx.x == 0) red[0] = a;
  }
  __syncthreads();
  const double nrm = sqrt(red[0]);
  if (nrm > 0.0)
    for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) v[j] = y[j] / nrm;
}
// one block: lab[i] = t[i] > (min t + max t) / 2
__global__ void k_label_by_midcut(const double* t, uint64_t cnt, uint8_t* lab) {
  __shared__ double lo_s[32], hi_s[32];
  double lo = INFINITY, hi = -INFINITY;
  for (uint64_t i = threadIdx.x; i < cnt; i += blockDim.x) { lo = fmin(lo, t[i]); hi = fmax(hi, t[i]); }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) { lo_s[threadIdx.x >> 5] = lo; hi_s[threadIdx.x >> 5] = hi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < blockDim.x / 32; ++w) { lo = fmin(lo, lo_s[w]); hi = fmax(hi, hi_s[w]); }
    lo_s[0] = lo;
    hi_s[0] = hi;
  }
  __syncthreads();
  const double cut = 0.5 * (lo_s[0] + hi_s[0]);
  for (uint64_t i = threadIdx.x; i < cnt; i += blockDim.x) lab[i] = t[i] > cut ? 1 : 0;
}

// Pass 2: warp per query slot; lanes own KP/32 survivors each; the `want`
// smallest (distance, id) keys are extracted in order. Slot v is point
// qlist[v] (qlist == nullptr: point v); candidates are indexed by slot, or by
// point id when by_row (then the fallback list records point ids too);
// want = min(k, size - 1) of its cluster (assign/sizes) or `fixed_want` when
// nonzero; list position offsets[point] or v * k when offsets == nullptr.
// Reference fp64 distances (ref_dist's j-ascending chain, bit for bit) of one
// query row to each lane's candidates. Candidate rows are staged through
// shared memory in 64-column chunks by coalesced warp-wide loads (128 bytes
// of one row per instruction), then each lane runs its own chain over its
// candidate's chunk (row stride 65: conflict-free). `tile` = 32 x 65 + 64
// floats per warp.
template <int PER>
__device__ __forceinline__ void warp_ref_dists(XPtr x, uint32_t d, XPtr qrow,
                                               const uint32_t (&iv)[PER], double (&dv)[PER],
                                               float* tile) {
  const int lane = threadIdx.x & 31;
  float* qt = tile + 32 * 65;
#pragma unroll
  for (int e = 0; e < PER; ++e) dv[e] = 0.0;
  for (uint32_t j0 = 0; j0 < d; j0 += 64) {
    const uint32_t w = min(64u, d - j0);
    __syncwarp();
    qt[lane] = lane < (int)w ? qrow[j0 + lane] : 0.f;
    qt[32 + lane] = 32 + lane < (int)w ? qrow[j0 + 32 + lane] : 0.f;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      __syncwarp();
      if (!x.bf) {
        // f32 rows: all 32 candidate rows' chunks in flight at once
        // (cp.async, no registers held), then one wait
        const float* xf = static_cast<const float*>(x.p);
        for (int c = 0; c < 32; ++c) {
          const uint32_t r = __shfl_sync(0xffffffffu, iv[e], c);
          if (r == 0xFFFFFFFFu) continue;  // warp-uniform
          const float* row = xf + (uint64_t)r * d + j0;
          float* t = tile + c * 65;
          if (lane < (int)w) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(t + lane)),
                         "l"(row + lane)
                         : "memory");
          } else {
            t[lane] = 0.f;
          }
          if (32 + lane < (int)w) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(t + 32 + lane)),
                         "l"(row + 32 + lane)
                         : "memory");
          } else {
            t[32 + lane] = 0.f;
          }
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
      } else {
#pragma unroll 4
        for (int c = 0; c < 32; ++c) {
          const uint32_t r = __shfl_sync(0xffffffffu, iv[e], c);
          if (r == 0xFFFFFFFFu) continue;  // warp-uniform
          const uint64_t row = (uint64_t)r * d + j0;
          tile[c * 65 + lane] = lane < (int)w ? x[row + lane] : 0.f;
          tile[c * 65 + 32 + lane] = 32 + lane < (int)w ? x[row + 32 + lane] : 0.f;
        }
      }
      __syncwarp();
      if (iv[e] != 0xFFFFFFFFu) {
        const float* mine = tile + lane * 65;
        double acc = dv[e];
        for (uint32_t j = 0; j < w; ++j) {
          const double t = __dsub_rn((double)qt[j], (double)mine[j]);
          acc = __dadd_rn(acc, __dmul_rn(t, t));
        }
        dv[e] = acc;
      }
    }
  }
#pragma unroll
  for (int e = 0; e < PER; ++e)
    if (iv[e] == 0xFFFFFFFFu) dv[e] = __longlong_as_double(0x7ff0000000000000ll);
}

constexpr int RR_WARP_FLOATS = 32 * 65 + 64;  // shared floats per warp of the re-rank

template <int KP>
__global__ void k_knn_rerank(XPtr x, uint32_t d, uint64_t nq,
                             const uint32_t* qlist, const uint32_t* assign, const uint32_t* sizes,
                             uint32_t k, uint32_t fixed_want, const uint32_t* cand_ids,
                             const float* cand_tau, const uint32_t* cand_cnt,
                             const uint32_t* offsets, uint32_t* out_nb, double* out_d,
                             uint32_t* fallback, uint32_t* n_fallback, double lb_factor,
                             int by_row) {
  constexpr int PER = KP / 32;
  const uint64_t v0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v0 >= nq) return;
  const uint64_t q = qlist ? qlist[v0] : v0;
  // by_row: candidate lists and the fallback record are indexed by point id
  const uint64_t v = by_row ? q : v0;
  const uint32_t want = fixed_want ? fixed_want : min(k, sizes[assign[q]] - 1);
  if (want == 0) return;
  const uint32_t c = cand_cnt[v];
  double dv[PER];
  uint32_t iv[PER];
#pragma unroll
  for (int e = 0; e < PER; ++e) {
    const int p = lane + 32 * e;  // slot
    iv[e] = p < (int)c ? cand_ids[v * KP + p] : 0xFFFFFFFFu;
  }
  extern __shared__ float rr_smem[];
  warp_ref_dists<PER>(x, d, x + q * d, iv, dv, rr_smem + (threadIdx.x >> 5) * RR_WARP_FLOATS);
  const uint64_t o = offsets ? (uint64_t)offsets[q] : v * k;
  double dk = 0.0;
  for (uint32_t r = 0; r < want; ++r) {
    double m = dv[0];
    uint32_t mi = iv[0];
    int me = 0;
#pragma unroll
    for (int e = 1; e < PER; ++e)
      if (key_less(dv[e], iv[e], m, mi)) { m = dv[e]; mi = iv[e]; me = e; }
    double wm = m;
    uint32_t wi = mi;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const double om = __shfl_xor_sync(0xffffffffu, wm, off);
      const uint32_t oi = __shfl_xor_sync(0xffffffffu, wi, off);
      if (key_less(om, oi, wm, wi)) { wm = om; wi = oi; }
    }
    if (mi == wi && wi != 0xFFFFFFFFu) {  // ids are unique: the owner retires it
#pragma unroll
      for (int e = 0; e < PER; ++e)
        if (e == me) { dv[e] = __longlong_as_double(0x7ff0000000000000ll); iv[e] = 0xFFFFFFFFu; }
    }
    if (lane == 0) {
      out_nb[o + r] = wi;
      if (out_d) out_d[o + r] = wm;
    }
    dk = wm;
  }
  // certificate (dk = the want-th exact distance among the survivors)
  const float t = cand_tau[v];
  // (every filter writes +inf when its list holds all candidates)
  const bool ok = isinf(t) || (double)t * lb_factor > dk;
  if (!ok && lane == 0) fallback[atomicAdd(n_fallback, 1u)] = (uint32_t)v;
}

// Launch the re-rank (8 warps per block, RR_WARP_FLOATS shared floats each).
template <int KP, typename... A>
void launch_rerank(uint64_t nwarps, cudaStream_t S, A... args) {
  const size_t smem = 8 * RR_WARP_FLOATS * sizeof(float);
  static bool attr = false;
  if (!attr) {
    NB_CUDA(cudaFuncSetAttribute(k_knn_rerank<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
    attr = true;
  }
  k_knn_rerank<KP><<<(unsigned)((nwarps * 32 + 255) / 256), 256, smem, S>>>(args...);
}

// Pass 3: one block per uncertified slot, exhaustive fp64 over its cluster
// (members[cl_beg[r] ..], or every point when members == nullptr); per-thread
// sorted top-`want`, merged by a block reduction. Slot / want / offsets as in
// pass 2.
template <int KMAX>
__global__ void __launch_bounds__(128) k_knn_exhaustive_t(
    XPtr x, uint32_t d, uint64_t n_all, const uint32_t* qlist,
    const uint32_t* assign, const uint32_t* members, const uint64_t* cl_beg,
    const uint32_t* sizes, uint32_t k, uint32_t fixed_want, const uint32_t* fallback,
    const uint32_t* offsets, uint32_t* out_nb, double* out_d) {
  __shared__ double sd[128 * 8];
  __shared__ uint32_t si[128 * 8];
  const uint32_t v = fallback[blockIdx.x];
  const uint32_t q = qlist ? qlist[v] : v;
  uint64_t size = n_all, beg = 0;
  if (members) {
    const uint32_t r = assign[q];
    size = sizes[r];
    beg = cl_beg[r];
  }
  const uint32_t want = fixed_want ? fixed_want : (uint32_t)umin64(k, size - 1);
  double bd[KMAX];
  uint32_t bi[KMAX];
  uint32_t cnt = 0;
  for (uint64_t t = threadIdx.x; t < size; t += blockDim.x) {
    const uint32_t j = members ? members[beg + t] : (uint32_t)t;
    if (j == q) continue;
    const double dd = ref_dist(x + (uint64_t)q * d, x + (uint64_t)j * d, d);
    if (cnt == want && !key_less(dd, j, bd[want - 1], bi[want - 1])) continue;
    uint32_t pos = cnt < want ? cnt : want - 1;
    while (pos > 0 && key_less(dd, j, bd[pos - 1], bi[pos - 1])) {
      bd[pos] = bd[pos - 1];
      bi[pos] = bi[pos - 1];
      --pos;
    }
    bd[pos] = dd;
    bi[pos] = j;
    if (cnt < want) ++cnt;
  }
  // merge: repeatedly take the global min of the per-thread list heads
  uint32_t head = 0;
  const uint64_t o = offsets ? (uint64_t)offsets[q] : (uint64_t)v * k;
  for (uint32_t r2 = 0; r2 < want; ++r2) {
    double val = head < cnt ? bd[head] : __longlong_as_double(0x7ff0000000000000ll);
    uint32_t vi = head < cnt ? bi[head] : 0xFFFFFFFFu;
    sd[threadIdx.x] = val;
    si[threadIdx.x] = vi;
    __syncthreads();
    for (int st = 64; st > 0; st >>= 1) {
      if ((int)threadIdx.x < st) {
        if (key_less(sd[threadIdx.x + st], si[threadIdx.x + st], sd[threadIdx.x], si[threadIdx.x])) {
          sd[threadIdx.x] = sd[threadIdx.x + st];
          si[threadIdx.x] = si[threadIdx.x + st];
        }
      }
      __syncthreads();
    }
    const uint32_t win = si[0];
    const double wd = sd[0];
    if (threadIdx.x == 0) {
      out_nb[o + r2] = win;
      if (out_d) out_d[o + r2] = wd;
    }
    if (head < cnt && bi[head] == win) ++head;
    __syncthreads();
  }
}

// the lists of the index build (k <= 64)
#define k_knn_exhaustive k_knn_exhaustive_t<64>

// Exact global top-k of every query in qlist over all n rows (reference fp64
// distance, (distance, id) order) for k beyond the filter's capacity
// (quality metrics with large k): one block per query.
void knn_exhaustive_rows(nomad_b200_ctx* ctx, XPtr x, uint64_t n, uint64_t d,
                         const uint32_t* qlist_d, uint32_t m, uint32_t k, uint32_t* out_ids_d) {
  cudaStream_t S = ctx->stream;
  if (k > 1024) fail(kParameter, "GPU exact kNN supports k <= 1024");
  DBuf<uint32_t> all(m);
  {
    std::vector<uint32_t> h(m);
    for (uint32_t i = 0; i < m; ++i) h[i] = i;
    NB_CUDA(cudaMemcpyAsync(all.p, h.data(), (uint64_t)m * 4, cudaMemcpyHostToDevice, S));
  }
  auto go = [&](auto kern) {
    kern<<<m, 128, 0, S>>>(x, (uint32_t)d, n, qlist_d, nullptr, nullptr, nullptr, nullptr, k, k,
                           all.p, nullptr, out_ids_d, nullptr);
  };
  if (k <= 64) go(k_knn_exhaustive_t<64>);
  else if (k <= 256) go(k_knn_exhaustive_t<256>);
  else go(k_knn_exhaustive_t<1024>);
  note_launch(ctx, "k_knn_exhaustive");
  NB_CUDA(cudaStreamSynchronize(S));
}

__global__ void k_knn_want(const uint32_t* assign, const uint32_t* sizes, uint64_t n, uint32_t k,
                           uint32_t* want) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = sizes[assign[i]];
    want[i] = min(k, s - 1);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) want[n] = 0;
}

__global__ void k_sizes2(const uint32_t* a, uint64_t n, uint32_t* sizes) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&sizes[a[i]], 1u);
}

}  // namespace

void knn_tc_candidates(nomad_b200_ctx* ctx, XPtr x, uint64_t n, uint64_t d,
                       const uint32_t* assign_d, uint32_t C, bool fp16, DBuf<uint32_t>& cand_ids,
                       DBuf<float>& cand_lb, DBuf<uint32_t>& cand_cnt, int* kp_out,
                       const std::vector<uint8_t>* own, int kp16, uint32_t max_qtiles = 0,
                       bool keep = false);

// Builds the graph into device buffers (offsets n+1, nb/dist offsets[n]).
struct KnnResult {
  DBuf<uint32_t> offsets, nb;
  DBuf<double> dist;
  uint64_t edges = 0;
  uint64_t fallbacks = 0;       // rows resolved by the exhaustive fp64 pass
  uint64_t tc_uncertified = 0;  // rows the tensor-core certificate did not settle
  uint64_t sub_certified = 0;   // of those, rows settled by the sub-cluster stage
};

// Concatenate the P partition lists of each query slot (slot-major, KP per
// partition) into one list of up to P * KP ids; the slot's bound is the
// smallest partition bound (+inf partitions hold all their candidates).
__global__ void k_merge_parts(uint32_t m, uint32_t P, uint32_t KP, const uint32_t* pid,
                              const float* plb, const uint32_t* pcnt, uint32_t* cid, float* clb,
                              uint32_t* ccnt) {
  const uint64_t v = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (v >= m) return;
  uint32_t c = 0;
  float lb = __int_as_float(0x7f800000);
  for (uint32_t p = 0; p < P; ++p) {
    const uint64_t e = v * P + p;
    const uint32_t cp = pcnt[e];
    for (uint32_t i = lane; i < cp; i += 32) cid[v * P * KP + c + i] = pid[e * KP + i];
    c += cp;
    lb = fminf(lb, plb[e]);
  }
  if (lane == 0) {
    ccnt[v] = c;
    clb[v] = lb;
  }
}

// ---- stage 1b (multi-blob clusters): exact kNN inside sub-clusters on the
// tensor cores + a geometric certificate against the other sub-clusters.

// Xr[i] = x[members[i]] (one cluster's rows, contiguous).
__global__ void k_gather_rows(XPtr x, const uint32_t* __restrict__ members,
                              uint64_t m, uint32_t d, float* __restrict__ xr) {
  const uint64_t N = m * d;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < N;
       e += (uint64_t)gridDim.x * blockDim.x)
    xr[e] = x[(uint64_t)members[e / d] * d + e % d];
}

__device__ __forceinline__ double dist_to(const float* __restrict__ row, const double* __restrict__ c,
                                          uint32_t d) {
  double acc = 0.0;
  for (uint32_t j = 0; j < d; ++j) {
    const double t = (double)row[j] - c[j];
    acc = fma(t, t, acc);
  }
  return sqrt(acc);
}

// radius[T] >= max over members of ||x - mu_T|| (bits of a positive double, atomicMax).
__global__ void k_sub_radius(const float* __restrict__ xr, uint64_t m, uint32_t d,
                             const uint32_t* __restrict__ sa, const double* __restrict__ cent,
                             double rel, unsigned long long* radius) {
  const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (v >= m) return;
  const uint32_t T = sa[v];
  const double r = dist_to(xr + v * d, cent + (uint64_t)T * d, d) * (1.0 + rel);
  atomicMax(radius + T, (unsigned long long)__double_as_longlong(r));
}

// Bisection helpers on index lists into the cluster's rows (heuristics only:
// they shape the partition, never the certificate).
// lab[i] = 1 if row idx[i] is closer to cen[1] than to cen[0]; sse[lab] += dist^2.
__global__ void k_assign2_idx(const float* __restrict__ xr, const uint32_t* __restrict__ idx,
                              uint64_t cnt, uint32_t d, const double* __restrict__ cen,
                              uint8_t* lab, double* sse) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  const float* row = xr + (uint64_t)idx[i] * d;
  const double a = dist_to(row, cen, d), b = dist_to(row, cen + d, d);
  const int l = b < a ? 1 : 0;
  lab[i] = (uint8_t)l;
  atomicAdd(sse + l, l ? b * b : a * a);
}
// Power-iteration passes for the segment's principal direction:
// t_i = (x_i - mu) . v ; y_j += sum_i t_i (x_ij - mu_j).
__global__ void k_proj_idx(const float* __restrict__ xr, const uint32_t* __restrict__ idx,
                           uint64_t cnt, uint32_t d, const double* __restrict__ mu,
                           const double* __restrict__ v, double* __restrict__ t) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  const float* row = xr + (uint64_t)idx[i] * d;
  double a = 0.0;
  for (uint32_t j = 0; j < d; ++j) a = fma((double)row[j] - mu[j], v[j], a);
  t[i] = a;
}
__global__ void k_backproj_idx(const float* __restrict__ xr, const uint32_t* __restrict__ idx,
                               uint64_t cnt, uint32_t d, const double* __restrict__ mu,
                               const double* __restrict__ t, double* __restrict__ y) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const uint64_t r0 = cnt * blockIdx.y / gridDim.y, r1 = cnt * (blockIdx.y + 1) / gridDim.y;
  double a = 0.0;
  for (uint64_t i = r0; i < r1; ++i) a = fma((double)xr[(uint64_t)idx[i] * d + j] - mu[j], t[i], a);
  atomicAdd(y + j, a);
}

// Row v (cluster-local) keeps its within-sub-cluster top-`want` (exact,
// tensor-core certified inside the sub-cluster) if every other sub-cluster T
// provably holds no closer point: for c in T, ||x_v - x_c|| >= D_T - R_T with
// D_T = ||x_v - mu_T||, R_T the sub-cluster radius, both computed in fp64 with
// a relative margin `rel`, and the reference's fp64 distance of the pair is
// >= that square times (1 - g64); sub-clusters of <= 64 rows are checked
// member by member instead. Certified rows are written back as complete
// candidate lists (global ids, +inf bound) so the re-rank reproduces them.
__global__ void k_sub_certify(const float* __restrict__ xr, uint64_t m, uint32_t d,
                              const uint32_t* __restrict__ sa, const double* __restrict__ cent,
                              const unsigned long long* __restrict__ radius,
                              const uint32_t* __restrict__ sizes_sub, uint32_t csub,
                              const uint32_t* __restrict__ seg_beg,
                              const uint32_t* __restrict__ seg_rows,
                              const uint8_t* __restrict__ open_sub, const uint32_t* __restrict__ ids2,
                              const double* __restrict__ d2, uint32_t k, uint32_t want,
                              const uint32_t* __restrict__ members, double rel, double g64,
                              uint32_t KP, uint32_t* cand_ids, float* cand_lb, uint32_t* cand_cnt,
                              unsigned long long* n_cert, uint32_t* cert_rows) {
  const uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (v >= m || open_sub[v]) return;
  if (ids2[v * k + want - 1] == 0xFFFFFFFFu) return;  // sub-cluster smaller than the list
  const double kth = d2[v * k + want - 1];
  const uint32_t S = sa[v];
  const float* row = xr + v * d;
  for (uint32_t T = 0; T < csub; ++T) {
    if (T == S || sizes_sub[T] == 0) continue;
    double gap;
    if (sizes_sub[T] <= 64) {  // small sub-cluster: its members directly
      double best = __longlong_as_double(0x7ff0000000000000ll);
      for (uint32_t e = 0; e < sizes_sub[T]; ++e) {
        const float* o = xr + (uint64_t)seg_rows[seg_beg[T] + e] * d;
        double acc = 0.0;
        for (uint32_t j = 0; j < d; ++j) {
          const double t = (double)row[j] - (double)o[j];
          acc = fma(t, t, acc);
        }
        best = fmin(best, acc);
      }
      gap = sqrt(best) * (1.0 - rel);
    } else {
      const double D = dist_to(row, cent + (uint64_t)T * d, d) * (1.0 - rel);
      const double R = __longlong_as_double((long long)radius[T]);
      gap = fmax(D - R, 0.0);
    }
    if (!(gap * gap * (1.0 - g64) * (1.0 - 1e-12) > kth)) return;
  }
  const uint64_t g = members[v];
  for (uint32_t i = 0; i < want; ++i) cand_ids[g * KP + i] = members[ids2[v * k + i]];
  cand_cnt[g] = want;
  cand_lb[g] = __int_as_float(0x7f800000);
  cert_rows[atomicAdd(n_cert, 1ull)] = (uint32_t)g;
}

__global__ void k_mark_rows(const uint32_t* list, uint32_t n, uint8_t* mask) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) mask[list[i]] = 1;
}

// FFMA certificate factor: every excluded candidate's reference distance is
// >= T / (1 + g32) * (1 - g64), T = the KP-th fp32 distance, with
// g32 = (d + 3) u32 for the fp32 chain and g64 = (d + 1) u64 for the
// reference's fp64 chain; rounded down generously.
double ffma_lb_factor(uint64_t d) {
  const double g32 = (double)(d + 3) * 0x1p-24 / (1.0 - (double)(d + 3) * 0x1p-24);
  const double g64 = (double)(d + 1) * 0x1p-53 / (1.0 - (double)(d + 1) * 0x1p-53);
  return (1.0 - g64) / (1.0 + g32) * (1.0 - 1e-12);
}

// Launch the FFMA filter over `sg` (ntiles query tiles in total).
void ffma_filter(nomad_b200_ctx* ctx, const float* x, uint64_t d, const uint32_t* members,
                 const uint32_t* qlist, const std::vector<FilterSeg>& sg, uint32_t ntiles, int kp,
                 int by_slot, uint32_t* cid, float* clb, uint32_t* ccnt) {
  cudaStream_t S = ctx->stream;
  DBuf<FilterSeg> sg_d(sg.size());
  NB_CUDA(cudaMemcpyAsync(sg_d.p, sg.data(), sg.size() * sizeof(FilterSeg), cudaMemcpyHostToDevice, S));
  const bool v4 = (d % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  const int cap = kp + CT / (kp <= 32 ? 2 : 4);
  const size_t smem = (size_t)2 * (QT + CT) * DK * 4 + (size_t)QT * cap * 8 + QT * 12;
  auto go = [&](auto kern) {
    NB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<ntiles, 256, smem, S>>>(x, (uint32_t)d, members, qlist, sg_d.p, (uint32_t)sg.size(),
                                   by_slot, cid, clb, ccnt, ffma_lb_factor(d));
  };
  if (kp == 32) {
    if (v4) go(k_knn_filter<32, true>); else go(k_knn_filter<32, false>);
  } else {
    if (v4) go(k_knn_filter<64, true>); else go(k_knn_filter<64, false>);
  }
  note_launch(ctx, "k_knn_filter");
  NB_CUDA(cudaStreamSynchronize(S));
}

// Stage 1b for one cluster (members[0..m)): returns the rows it certified.
constexpr uint64_t kBisectSample = 16384;  // rows that shape a bisection (knn subcluster_stage)

uint64_t subcluster_stage(nomad_b200_ctx* ctx, XPtr x, uint64_t d, const uint32_t* members,
                          uint64_t m, uint32_t k, int KP, DBuf<uint32_t>& cid, DBuf<float>& clb,
                          DBuf<uint32_t>& ccnt, std::vector<uint32_t>& cert_out) {
  cudaStream_t S = ctx->stream;
  const bool dbg = std::getenv("NOMAD_B200_DEBUG_KNN") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!dbg) return;
    NB_CUDA(cudaStreamSynchronize(S));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "    1b %-22s %7.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  DBuf<float> xr(m * d);
  k_gather_rows<<<ctx->sm_count * 8, 256, 0, S>>>(x, members, m, (uint32_t)d, xr.p);
  note_launch(ctx, "k_gather_rows");
  // Sub-clusters by recursive bisection: a segment is split by 2-means
  // (principal-direction initialisation, then Lloyd steps) when the split
  // removes >= 3 % of the segment's squared error about its mean (in high
  // dimension, halving one Gaussian blob removes ~0.1 %, separating blobs far
  // more), or when one side is a small far group (< 5 %: a fragment of
  // another blob, peeled off); otherwise it is kept whole. Well-separated blobs end up one per
  // sub-cluster (a split blob would leave its points without a geometric
  // certificate, a merged pair without a tight tensor-core one). Any
  // partition is valid for the certificate; this only decides how many rows
  // it settles.
  const double rel = (double)(d + 8) * 0x1p-52;
  // 2-means of one index list, initialised by its principal direction
  // (PDDP), then Lloyd steps, all on the device; returns false when the split
  // removes < 3 % of the squared error about the mean (one blob) or is
  // degenerate.
  // bisection scratch, sized for the whole cluster once (cudaMalloc / cudaFree
  // per bisection would dominate the stage)
  DBuf<uint32_t> ix(m), ixs(std::min<uint64_t>(m, kBisectSample));
  DBuf<uint8_t> blab(m);
  DBuf<double> cen(2 * d), sums(2 * d), sse(4), vd(d), yd(d), td(m);
  DBuf<unsigned long long> cnts(2);
  auto bisect = [&](const std::vector<uint32_t>& seg, std::vector<uint32_t>& a0,
                    std::vector<uint32_t>& a1) -> bool {
    const uint64_t c = seg.size();
    NB_CUDA(cudaMemcpyAsync(ix.p, seg.data(), c * 4, cudaMemcpyHostToDevice, S));
    const unsigned gb = (unsigned)((c + 127) / 128);
    const dim3 gs((unsigned)((d + 127) / 128), 64);
    auto label_means = [&](const uint32_t* idx, uint64_t cnt, const uint8_t* l) {
      NB_CUDA(cudaMemsetAsync(sums.p, 0, 2 * d * 8, S));
      NB_CUDA(cudaMemsetAsync(cnts.p, 0, 16, S));
      k_label_sums<<<gs, 128, 0, S>>>(xr.p, idx, cnt, (uint32_t)d, l, sums.p, cnts.p);
      k_means_from_sums<<<8, 256, 0, S>>>(sums.p, cnts.p, (uint32_t)d, cen.p);
    };
    // mean (cen[0]) and the parent error about it (sse[2..3], labels all 0)
    label_means(ix.p, c, nullptr);
    NB_CUDA(cudaMemcpyAsync(cen.p + d, cen.p, d * 8, cudaMemcpyDeviceToDevice, S));
    NB_CUDA(cudaMemsetAsync(sse.p, 0, 32, S));
    k_assign2_idx<<<gb, 128, 0, S>>>(xr.p, ix.p, c, (uint32_t)d, cen.p, blab.p, sse.p + 2);
    // The split direction and centroids come from an evenly strided sample of
    // at most kBisectSample rows (they shape the partition, never the
    // certificate); the split itself labels every row.
    uint64_t cs = c;
    const uint32_t* is = ix.p;
    if (c > 2 * kBisectSample) {
      const uint64_t stride = c / kBisectSample;
      std::vector<uint32_t> sm;
      sm.reserve(kBisectSample);
      for (uint64_t i = 0; i < c && sm.size() < kBisectSample; i += stride) sm.push_back(seg[i]);
      cs = sm.size();
      NB_CUDA(cudaMemcpyAsync(ixs.p, sm.data(), cs * 4, cudaMemcpyHostToDevice, S));
      is = ixs.p;
    }
    const unsigned gbs = (unsigned)((cs + 127) / 128);
    // principal direction (5 power steps from a fixed start), cut across it at
    // the middle of the projected range (separates a far fragment at one end
    // as well as two groups of blobs), then two Lloyd steps
    {
      std::vector<double> vh(d);
      HostRng g(0x70646470 /* "pddp" */);
      for (auto& e : vh) e = g.gaussian();
      NB_CUDA(cudaMemcpyAsync(yd.p, vh.data(), d * 8, cudaMemcpyHostToDevice, S));
      for (int it = 0; it < 5; ++it) {
        k_normalize<<<1, 256, 0, S>>>(yd.p, (uint32_t)d, vd.p);
        k_proj_idx<<<gbs, 128, 0, S>>>(xr.p, is, cs, (uint32_t)d, cen.p, vd.p, td.p);
        NB_CUDA(cudaMemsetAsync(yd.p, 0, d * 8, S));
        k_backproj_idx<<<gs, 128, 0, S>>>(xr.p, is, cs, (uint32_t)d, cen.p, td.p, yd.p);
      }
      k_label_by_midcut<<<1, 1024, 0, S>>>(td.p, cs, blab.p);
    }
    for (int it = 0; it < 2; ++it) {
      label_means(is, cs, blab.p);
      NB_CUDA(cudaMemsetAsync(sse.p, 0, 16, S));
      k_assign2_idx<<<gbs, 128, 0, S>>>(xr.p, is, cs, (uint32_t)d, cen.p, blab.p, sse.p);
    }
    if (is != ix.p) {  // every row against the sample's two centroids
      NB_CUDA(cudaMemsetAsync(sse.p, 0, 16, S));
      k_assign2_idx<<<gb, 128, 0, S>>>(xr.p, ix.p, c, (uint32_t)d, cen.p, blab.p, sse.p);
    }
    note_launch(ctx, "k_bisect");
    std::vector<uint8_t> lh(c);
    double ss[4];
    NB_CUDA(cudaMemcpyAsync(lh.data(), blab.p, c, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaMemcpyAsync(ss, sse.p, 32, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    const double parent = ss[2] + ss[3];
    a0.clear();
    a1.clear();
    for (uint64_t i = 0; i < c; ++i) (lh[i] ? a1 : a0).push_back(seg[i]);
    if (a0.empty() || a1.empty()) return false;
    if (std::getenv("NOMAD_B200_DEBUG_KNN"))
      std::fprintf(stderr, "  bisect %llu rows: parent %.4g split %.4g (%zu / %zu)\n",
                   (unsigned long long)c, parent, ss[0] + ss[1], a0.size(), a1.size());
    // a small far group (a fragment of another blob) is peeled off whatever
    // the error reduction; a balanced split must remove >= 3 %
    if (std::min(a0.size(), a1.size()) * 20 < c) return true;
    return ss[0] + ss[1] < 0.97 * parent;
  };
  std::vector<std::vector<uint32_t>> done, work;
  {
    std::vector<uint32_t> all(m);
    for (uint64_t i = 0; i < m; ++i) all[i] = (uint32_t)i;
    work.push_back(std::move(all));
  }
  while (!work.empty() && done.size() + work.size() < 256) {
    std::vector<uint32_t> seg = std::move(work.back());
    work.pop_back();
    std::vector<uint32_t> a0, a1;
    if (seg.size() < 2 || !bisect(seg, a0, a1)) {
      done.push_back(std::move(seg));
      continue;
    }
    work.push_back(std::move(a0));
    work.push_back(std::move(a1));
  }
  for (auto& w : work) done.push_back(std::move(w));
  lap("gather + bisection");
  const uint32_t csub = (uint32_t)done.size();
  if (std::getenv("NOMAD_B200_DEBUG_KNN"))
    std::fprintf(stderr, "subcluster bisection: m=%llu -> %u segments\n", (unsigned long long)m, csub);
  if (csub < 2) return 0;
  // labels, sizes and exact segment means (any centre is valid)
  std::vector<uint32_t> lab(m), szh(csub);
  for (uint32_t t = 0; t < csub; ++t) {
    szh[t] = (uint32_t)done[t].size();
    for (uint32_t i : done[t]) lab[i] = t;
  }
  DBuf<uint32_t> sa(m), ssz(csub), od, segb;
  DBuf<double> sc((uint64_t)csub * d);
  NB_CUDA(cudaMemcpyAsync(sa.p, lab.data(), m * 4, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(ssz.p, szh.data(), csub * 4, cudaMemcpyHostToDevice, S));
  {
    std::vector<uint32_t> order;
    std::vector<uint64_t> beg, cnt;
    std::vector<uint32_t> ids;
    for (uint32_t t = 0; t < csub; ++t) {
      beg.push_back(order.size());
      cnt.push_back(done[t].size());
      ids.push_back(t);
      std::vector<uint32_t> sorted = done[t];
      std::sort(sorted.begin(), sorted.end());
      order.insert(order.end(), sorted.begin(), sorted.end());
    }
    od.alloc(m);
    NB_CUDA(cudaMemcpyAsync(od.p, order.data(), m * 4, cudaMemcpyHostToDevice, S));
    fast_column_means(ctx, xr.p, d, od.p, beg, cnt, ids, sc.p);  // any fixed centre
    std::vector<uint32_t> b32(beg.begin(), beg.end());
    segb.alloc(csub);
    NB_CUDA(cudaMemcpyAsync(segb.p, b32.data(), csub * 4, cudaMemcpyHostToDevice, S));
    NB_CUDA(cudaStreamSynchronize(S));
  }
  DBuf<uint32_t> cid2, ccnt2;
  DBuf<float> clb2;
  int KP2 = 0;
  lap("labels + means");
  knn_tc_candidates(ctx, xr.p, m, d, sa.p, csub, true, cid2, clb2, ccnt2, &KP2, nullptr, 64);
  lap("tensor-core lists");
  const uint32_t want = (uint32_t)std::min<uint64_t>(k, m - 1);
  DBuf<uint32_t> ids2(m * k), fb2(m), nfb2(1);
  DBuf<double> d2(m * k);
  NB_CUDA(cudaMemsetAsync(nfb2.p, 0, 4, S));
  NB_CUDA(cudaMemsetAsync(ids2.p, 0xFF, m * k * 4, S));
  auto go2 = [&](auto kp) {
    launch_rerank<decltype(kp)::value>(m, S, XPtr(xr.p), (uint32_t)d, m,
                                       (const uint32_t*)nullptr, (const uint32_t*)nullptr,
                                       (const uint32_t*)nullptr, k, want, (const uint32_t*)cid2.p,
                                       (const float*)clb2.p, (const uint32_t*)ccnt2.p,
                                       (const uint32_t*)nullptr, ids2.p, d2.p, fb2.p, nfb2.p, 1.0,
                                       0);
  };
  if (KP2 == 32) go2(std::integral_constant<int, 32>{}); else go2(std::integral_constant<int, 64>{});
  note_launch(ctx, "k_knn_rerank");
  uint32_t nf2 = 0;
  NB_CUDA(cudaMemcpyAsync(&nf2, nfb2.p, 4, cudaMemcpyDeviceToHost, S));
  NB_CUDA(cudaStreamSynchronize(S));
  lap("re-rank");
  DBuf<uint8_t> open(m);
  NB_CUDA(cudaMemsetAsync(open.p, 0, m, S));
  if (nf2) {
    k_mark_rows<<<(nf2 + 255) / 256, 256, 0, S>>>(fb2.p, nf2, open.p);
    note_launch(ctx, "k_mark_rows");
  }
  const double g64 = (double)(d + 1) * 0x1p-53 * 2;
  DBuf<unsigned long long> rad(csub), ncert(1);
  DBuf<uint32_t> crows(m);
  NB_CUDA(cudaMemsetAsync(rad.p, 0, csub * 8, S));
  NB_CUDA(cudaMemsetAsync(ncert.p, 0, 8, S));
  const unsigned mb = (unsigned)((m + 127) / 128);
  k_sub_radius<<<mb, 128, 0, S>>>(xr.p, m, (uint32_t)d, sa.p, sc.p, rel, rad.p);
  note_launch(ctx, "k_sub_radius");
  k_sub_certify<<<mb, 128, 0, S>>>(xr.p, m, (uint32_t)d, sa.p, sc.p, rad.p, ssz.p, csub, segb.p,
                                   od.p, open.p,
                                   ids2.p, d2.p, k, want, members, rel, g64, (uint32_t)KP, cid.p,
                                   clb.p, ccnt.p, ncert.p, crows.p);
  note_launch(ctx, "k_sub_certify");
  unsigned long long nc = 0;
  NB_CUDA(cudaMemcpyAsync(&nc, ncert.p, 8, cudaMemcpyDeviceToHost, S));
  NB_CUDA(cudaStreamSynchronize(S));
  lap("radius + certify");
  if (nc) {
    const size_t o = cert_out.size();
    cert_out.resize(o + nc);
    NB_CUDA(cudaMemcpy(cert_out.data() + o, crows.p, nc * 4, cudaMemcpyDeviceToHost));
  }
  if (dbg) {
    const auto t0 = std::chrono::steady_clock::now();
    DBuf<float> probe(m * d);  // debug: cost of one cluster-sized allocation + free (cached)
    probe.release();
    std::fprintf(stderr, "    1b alloc+free %zu MB: %.1f ms\n", (size_t)(m * d * 4 >> 20),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  if (std::getenv("NOMAD_B200_DEBUG_KNN")) {
    std::fprintf(stderr, "subcluster stage: m=%llu csub=%u open-within=%u certified=%llu sizes:",
                 (unsigned long long)m, csub, nf2, nc);
    for (uint32_t t = 0; t < csub; ++t) std::fprintf(stderr, " %u", szh[t]);
    std::vector<unsigned long long> rh(csub);
    NB_CUDA(cudaMemcpy(rh.data(), rad.p, csub * 8, cudaMemcpyDeviceToHost));
    std::fprintf(stderr, " radii:");
    for (uint32_t t = 0; t < csub; ++t) { double r; std::memcpy(&r, &rh[t], 8); std::fprintf(stderr, " %.1f", r); }
    std::fprintf(stderr, "\n");
  }
  return nc;
}

// bf16 rows for the FFMA filter: rows ids[i] (or lo + i) widened to f32.
__global__ void k_widen_rows(XPtr x, const uint32_t* ids, uint64_t lo, uint64_t rows, uint32_t d,
                             float* out) {
  const uint64_t N = rows * d;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < N;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = e / d, j = e % d;
    out[e] = x[(ids ? (uint64_t)ids[r] : lo + r) * d + j];
  }
}

// Slot-indexed lists of one cluster's widened-row filter -> row-indexed
// lists with global ids (members of the cluster, ascending).
__global__ void k_scatter_slots(uint32_t qn, uint32_t KP, const uint32_t* qglob,
                                const uint32_t* cmem, const uint32_t* tid, const float* tlb,
                                const uint32_t* tcnt, uint32_t* cid, float* clb, uint32_t* ccnt) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= qn) return;
  const uint64_t gq = qglob[v];
  const uint32_t c = tcnt[v];
  for (uint32_t e = 0; e < c; ++e) cid[gq * KP + e] = cmem[tid[(uint64_t)v * KP + e]];
  ccnt[gq] = c;
  clb[gq] = tlb[v];
}

// own: nullptr = every cluster; else own[r] != 0 for the clusters whose lists
// are built (multi-GPU: the clusters of this rank's shards); rows of the other
// clusters get empty lists.
void build_knn_exact(nomad_b200_ctx* ctx, XPtr x, uint64_t n, uint64_t d,
                     const uint32_t* assign_d, uint32_t C, uint32_t k, KnnResult& R,
                     int mode, const std::vector<uint8_t>* own) {
  cudaStream_t S = ctx->stream;
  if (k < 1) fail(kParameter, "k must be >= 1");
  if (k > 56) fail(kParameter, "k > 56 is not supported by the exact kNN build");
  DBuf<uint32_t> sizes(C);
  NB_CUDA(cudaMemsetAsync(sizes.p, 0, C * 4, S));
  k_sizes2<<<(unsigned)std::min<uint64_t>(4096, (n + 255) / 256), 256, 0, S>>>(assign_d, n, sizes.p);
  note_launch(ctx, "k_sizes");
  // list lengths: min(k, size - 1), 0 outside the owned clusters
  DBuf<uint32_t> sizes_eff;
  const uint32_t* sizes_want = sizes.p;
  if (own) {
    std::vector<uint32_t> sh(C);
    NB_CUDA(cudaMemcpyAsync(sh.data(), sizes.p, C * 4, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    for (uint32_t r = 0; r < C; ++r)
      if (!(*own)[r]) sh[r] = 1;
    sizes_eff.alloc(C);
    NB_CUDA(cudaMemcpyAsync(sizes_eff.p, sh.data(), C * 4, cudaMemcpyHostToDevice, S));
    sizes_want = sizes_eff.p;
  }
  // offsets = exclusive scan of min(k, size-1) (knn.hpp:77-83)
  DBuf<uint32_t> want(n + 1);
  k_knn_want<<<(unsigned)std::min<uint64_t>(4096, (n + 255) / 256), 256, 0, S>>>(assign_d, sizes_want, n, k, want.p);
  note_launch(ctx, "k_knn_want");
  R.offsets.alloc(n + 1);
  size_t tmp = 0;
  NB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, want.p, R.offsets.p, (int64_t)(n + 1), S));
  DBuf<uint8_t> tb(tmp + 1);
  NB_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, tmp, want.p, R.offsets.p, (int64_t)(n + 1), S));
  note_launch(ctx, "cub_exclusive_sum");
  uint32_t edges = 0;
  NB_CUDA(cudaMemcpyAsync(&edges, R.offsets.p + n, 4, cudaMemcpyDeviceToHost, S));
  // members per cluster, ascending id (knn.hpp:70-72)
  DBuf<uint32_t> mem;
  std::vector<uint64_t> off;
  group_by_label(ctx, assign_d, n, C, mem, off);
  R.edges = edges;
  R.nb.alloc(std::max<uint64_t>(edges, 1));
  R.dist.alloc(std::max<uint64_t>(edges, 1));
  // whole-cluster segments (queries = candidates = the cluster's members)
  std::vector<FilterSeg> segs;
  uint32_t tiles = 0;
  for (uint32_t r = 0; r < C; ++r) {
    const uint32_t sz = (uint32_t)(off[r + 1] - off[r]);
    if (sz < 2 || (own && !(*own)[r])) continue;
    segs.push_back(FilterSeg{off[r], off[r], sz, sz, tiles, 0});
    tiles += (sz + QT - 1) / QT;
  }
  if (tiles == 0) {
    NB_CUDA(cudaStreamSynchronize(S));
    return;
  }
  int KP = k <= 24 ? 32 : 64;
  DBuf<uint32_t> cid, ccnt;
  DBuf<float> clb;  // per-row lower bound on every excluded reference distance
  // Re-rank the listed rows (device list, m rows; candidates indexed by row)
  // and return the rows whose certificate failed. The first pass walks every
  // row in cluster order (mem), so concurrently re-ranked queries share their
  // candidates' rows in L2; later passes touch only the rows a stage changed.
  DBuf<uint32_t> fb(n), nfb(1);
  auto rerank_rows = [&](const uint32_t* rows_d, uint64_t m) {
    std::vector<uint32_t> out;
    if (!m) return out;
    NB_CUDA(cudaMemsetAsync(nfb.p, 0, 4, S));
    auto go = [&](auto kp) {
      launch_rerank<decltype(kp)::value>(m, S, x, (uint32_t)d, m, rows_d, assign_d, sizes_want, k,
                                         0u, (const uint32_t*)cid.p, (const float*)clb.p,
                                         (const uint32_t*)ccnt.p, (const uint32_t*)R.offsets.p,
                                         R.nb.p, R.dist.p, fb.p, nfb.p, 1.0, 1);
    };
    if (KP == 32) go(std::integral_constant<int, 32>{}); else go(std::integral_constant<int, 64>{});
    note_launch(ctx, "k_knn_rerank");
    uint32_t nf = 0;
    NB_CUDA(cudaMemcpyAsync(&nf, nfb.p, 4, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    out.resize(nf);
    if (nf) NB_CUDA(cudaMemcpy(out.data(), fb.p, nf * 4, cudaMemcpyDeviceToHost));
    return out;
  };
  auto upload_rows = [&](const std::vector<uint32_t>& rows, DBuf<uint32_t>& dst) {
    dst.alloc(std::max<size_t>(rows.size(), 1));
    if (!rows.empty())
      NB_CUDA(cudaMemcpyAsync(dst.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, S));
  };
  // FFMA certified filter over segments of clusters (queries qh[sg.qbeg ..]
  // are global ids, candidates the cluster's members). bf16 rows: each
  // cluster's rows are widened into an f32 scratch and filtered in local
  // indices (self excluded there), then scattered back to global ids.
  std::vector<uint32_t> mem_h;
  auto ffma_segments = [&](const std::vector<FilterSeg>& sg, uint32_t ntiles,
                           const std::vector<uint32_t>& qh, const uint32_t* ql_d) {
    if (!x.bf) {
      ffma_filter(ctx, static_cast<const float*>(x.p), d, mem.p, ql_d, sg, ntiles, KP, 0, cid.p,
                  clb.p, ccnt.p);
      return;
    }
    if (mem_h.empty()) {
      mem_h.resize(n);
      NB_CUDA(cudaMemcpy(mem_h.data(), mem.p, n * 4, cudaMemcpyDeviceToHost));
    }
    for (const FilterSeg& g : sg) {
      const uint64_t sz = g.size, qn = g.qn;
      DBuf<float> scr(sz * d);
      k_widen_rows<<<ctx->sm_count * 8, 256, 0, S>>>(x, mem.p + g.beg, 0, sz, (uint32_t)d, scr.p);
      note_launch(ctx, "k_widen_rows");
      std::vector<uint32_t> lq(qn), gq(qn);
      for (uint64_t v = 0; v < qn; ++v) {
        gq[v] = qh[g.qbeg + v];
        lq[v] = (uint32_t)(std::lower_bound(mem_h.begin() + g.beg, mem_h.begin() + g.beg + sz,
                                            gq[v]) - (mem_h.begin() + g.beg));
      }
      DBuf<uint32_t> lq_d, gq_d, tid(qn * KP), tcnt(qn);
      DBuf<float> tlb(qn);
      upload_rows(lq, lq_d);
      upload_rows(gq, gq_d);
      const std::vector<FilterSeg> one{FilterSeg{0, 0, (uint32_t)sz, (uint32_t)qn, 0, 0}};
      ffma_filter(ctx, scr.p, d, nullptr, lq_d.p, one, (uint32_t)((qn + QT - 1) / QT), KP, 1,
                  tid.p, tlb.p, tcnt.p);
      k_scatter_slots<<<(unsigned)((qn + 127) / 128), 128, 0, S>>>(
          (uint32_t)qn, (uint32_t)KP, gq_d.p, mem.p + g.beg, tid.p, tlb.p, tcnt.p, cid.p, clb.p,
          ccnt.p);
      note_launch(ctx, "k_scatter_slots");
      NB_CUDA(cudaStreamSynchronize(S));
    }
  };
  // open \ settled, then + the settled rows that failed again
  auto update_open = [&](std::vector<uint32_t>& open, std::vector<uint32_t> settled,
                         const std::vector<uint32_t>& failed) {
    std::sort(settled.begin(), settled.end());
    std::vector<uint32_t> rest;
    for (uint32_t q : open)
      if (!std::binary_search(settled.begin(), settled.end(), q)) rest.push_back(q);
    rest.insert(rest.end(), failed.begin(), failed.end());
    open.swap(rest);
  };

  const bool tc = (mode == NOMAD_B200_KNN_BF16) || (mode == NOMAD_B200_KNN_EXACT && k <= 56);
  std::vector<uint32_t> open;
  const bool dbg = std::getenv("NOMAD_B200_DEBUG_KNN") != nullptr;
  auto t_stage = std::chrono::steady_clock::now();
  auto stage_done = [&](const char* what) {
    if (!dbg) return;
    NB_CUDA(cudaStreamSynchronize(S));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "knn stage %-28s %8.1f ms, open rows %zu\n", what,
                 std::chrono::duration<double, std::milli>(now - t_stage).count(), open.size());
    t_stage = now;
  };
  if (tc) {
    // stage 1: tensor-core filter (bf16 fast / fp16 certified)
    if (mode == NOMAD_B200_KNN_BF16 && k > 24) fail(kParameter, "bf16 kNN mode supports k <= 24");
    // certified lists: top-32 in the main stage when k <= 24 (measured: 39 % fewer SM
    // cycles than top-64 at 10M, same rows certified); top-64 inside sub-clusters
    // (stage 1b), where the certificate needs the wider margin.
    // NOMAD_B200_EXACT_KP=64 restores top-64 in the main stage.
    static const bool force64 = [] {
      const char* e = std::getenv("NOMAD_B200_EXACT_KP");
      return e && std::atoi(e) == 64;
    }();
    const int kp_main = (k <= 24 && !force64) ? 32 : 64;
    if (mode == NOMAD_B200_KNN_EXACT && C > 1) {
      // Probe: the first query tile (128 rows) of every cluster through the
      // certified filter + re-rank. A large cluster where most probe rows
      // stay uncertified spans several blobs (its centred norms dwarf its
      // neighbour distances): the main pass skips it and its rows go straight
      // to the sub-cluster stage, which the main pass could not spare them.
      // A wrong guess only moves rows between exact stages.
      knn_tc_candidates(ctx, x, n, d, assign_d, C, true, cid, clb, ccnt, &KP, own, kp_main, 1);
      std::vector<uint32_t> probe;
      std::vector<uint64_t> pcount(C, 0);
      {
        std::vector<uint32_t> mh(n);
        NB_CUDA(cudaMemcpy(mh.data(), mem.p, n * 4, cudaMemcpyDeviceToHost));
        for (uint32_t r = 0; r < C; ++r) {
          const uint64_t sz = off[r + 1] - off[r];
          if (sz < 2 || (own && !(*own)[r])) continue;
          const uint64_t m = std::min<uint64_t>(sz, 128);
          pcount[r] = m;
          probe.insert(probe.end(), mh.begin() + off[r], mh.begin() + off[r] + m);
        }
      }
      std::vector<uint32_t> failed;
      if (!probe.empty()) {
        DBuf<uint32_t> pd;
        upload_rows(probe, pd);
        failed = rerank_rows(pd.p, probe.size());
      }
      std::vector<uint64_t> pfail(C, 0);
      {
        std::vector<uint32_t> ah0(n);
        NB_CUDA(cudaMemcpy(ah0.data(), assign_d, n * 4, cudaMemcpyDeviceToHost));
        for (uint32_t q : failed) ++pfail[ah0[q]];
      }
      std::vector<uint8_t> own2(C, 1);
      uint32_t skipped = 0;
      for (uint32_t r = 0; r < C; ++r) {
        if (own && !(*own)[r]) own2[r] = 0;
        const uint64_t sz = off[r + 1] - off[r];
        if (sz >= 1024 && pcount[r] && pfail[r] * 2 >= pcount[r]) {
          own2[r] = 0;
          ++skipped;
        }
      }
      stage_done("probe");
      if (dbg) std::fprintf(stderr, "knn probe: %u multi-blob clusters skip the main pass\n", skipped);
      knn_tc_candidates(ctx, x, n, d, assign_d, C, true, cid, clb, ccnt, &KP, &own2, kp_main, 0,
                        true);
    } else {
      knn_tc_candidates(ctx, x, n, d, assign_d, C, mode == NOMAD_B200_KNN_EXACT, cid, clb, ccnt,
                        &KP, own, kp_main);
    }
    stage_done("tensor-core candidates");
    open = rerank_rows(std::getenv("NOMAD_B200_KNN_IDORDER") ? nullptr : mem.p, n);
    R.tc_uncertified = open.size();
    stage_done("re-rank");
    std::vector<uint32_t> ah;
    auto fail_count = [&](std::vector<uint64_t>& fail_per) {
      if (ah.empty()) {
        ah.resize(n);
        NB_CUDA(cudaMemcpy(ah.data(), assign_d, n * 4, cudaMemcpyDeviceToHost));
      }
      fail_per.assign(C, 0);
      for (uint32_t q : open) ++fail_per[ah[q]];
    };
    if (!open.empty() && mode == NOMAD_B200_KNN_EXACT) {
      // stage 1b: clusters where many rows failed the tensor-core certificate
      // (centred norms >> neighbour distances: the cluster spans several
      // blobs) are split into sub-clusters; exact lists inside each
      // sub-cluster come from the certified tensor-core filter on the
      // sub-cluster's own centring, and a row keeps its list when no other
      // sub-cluster can hold a closer point (k_sub_certify).
      std::vector<uint64_t> fail_per;
      fail_count(fail_per);
      std::vector<uint32_t> cert;
      for (uint32_t r = 0; r < C; ++r) {
        const uint64_t sz = off[r + 1] - off[r];
        if (sz < 1024 || own && !(*own)[r] || fail_per[r] * 16 < sz) continue;
        const auto t_sc = std::chrono::steady_clock::now();
        subcluster_stage(ctx, x, d, mem.p + off[r], sz, k, KP, cid, clb, ccnt, cert);
        if (std::getenv("NOMAD_B200_DEBUG_KNN"))
          std::fprintf(stderr, "    1b cluster %u: %.1f ms in total\n", r,
                       std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_sc).count());
      }
      R.sub_certified = cert.size();
      stage_done("sub-cluster stage");
      if (!cert.empty()) {
        DBuf<uint32_t> cd;
        upload_rows(cert, cd);
        const std::vector<uint32_t> again = rerank_rows(cd.p, cert.size());
        update_open(open, cert, again);
      }
      stage_done("re-rank (sub-cluster rows)");
    }
    if (!open.empty() && mode == NOMAD_B200_KNN_EXACT) {
      // stage 2: rows still open (both certificates failed) get the FFMA
      // filter against their whole cluster, whose error is relative to the
      // distance itself; clusters with a handful of open rows go straight to
      // the exhaustive pass
      std::vector<uint64_t> fail_per;
      fail_count(fail_per);
      std::vector<uint64_t> qoff(C + 1, 0);
      for (uint32_t r = 0; r < C; ++r) qoff[r + 1] = qoff[r] + (fail_per[r] >= 16 ? fail_per[r] : 0);
      std::vector<uint32_t> qh(qoff[C]);
      std::vector<uint64_t> fill(qoff.begin(), qoff.end() - 1);
      std::vector<uint32_t> sorted_open(open);
      std::sort(sorted_open.begin(), sorted_open.end());
      for (uint32_t q : sorted_open)
        if (fail_per[ah[q]] >= 16) qh[fill[ah[q]]++] = q;
      std::vector<FilterSeg> sg;
      uint32_t nt = 0;
      for (uint32_t r = 0; r < C; ++r) {
        const uint64_t sz = off[r + 1] - off[r];
        const uint64_t qn = qoff[r + 1] - qoff[r];
        if (sz < 2 || qn == 0) continue;
        sg.push_back(FilterSeg{off[r], qoff[r], (uint32_t)sz, (uint32_t)qn, nt, 0});
        nt += (uint32_t)((qn + QT - 1) / QT);
      }
      if (nt) {
        DBuf<uint32_t> ql;
        upload_rows(qh, ql);
        ffma_segments(sg, nt, qh, ql.p);
        const std::vector<uint32_t> again = rerank_rows(ql.p, qh.size());
        update_open(open, qh, again);
      }
      stage_done("FFMA stage");
    }
  } else {
    cid.alloc(n * (uint64_t)KP);
    ccnt.alloc(n);
    clb.alloc(n);
    NB_CUDA(cudaMemsetAsync(ccnt.p, 0, n * 4, S));
    if (x.bf) {
      std::vector<uint32_t> all(n);
      NB_CUDA(cudaMemcpy(all.data(), mem.p, n * 4, cudaMemcpyDeviceToHost));
      ffma_segments(segs, tiles, all, mem.p);
    } else {
      ffma_segments(segs, tiles, {}, mem.p);
    }
    open = rerank_rows(mem.p, n);
  }
  // stage 3: exhaustive fp64 for whatever is still uncertified
  R.fallbacks = open.size();
  if (!open.empty()) {
    std::vector<uint64_t> cb(C);
    for (uint32_t r = 0; r < C; ++r) cb[r] = off[r];
    DBuf<uint64_t> cb_d(C);
    NB_CUDA(cudaMemcpyAsync(cb_d.p, cb.data(), C * 8, cudaMemcpyHostToDevice, S));
    DBuf<uint32_t> od;
    upload_rows(open, od);
    k_knn_exhaustive<<<(unsigned)open.size(), 128, 0, S>>>(x, (uint32_t)d, n, nullptr, assign_d,
                                                           mem.p, cb_d.p, sizes.p, k, 0u, od.p,
                                                           R.offsets.p, R.nb.p, R.dist.p);
    note_launch(ctx, "k_knn_exhaustive");
  }
  NB_CUDA(cudaStreamSynchronize(S));
}

// Partition `part` of a widened-chunk filter: candidate ids are scratch rows
// (off_m + local row) -> global ids lo + local row; the query itself (it is
// not excluded inside the scratch) is dropped. The partition bound stays
// valid (every excluded candidate is >= it).
__global__ void k_remap_part(uint32_t m, uint32_t P, uint32_t KP, uint32_t part, uint32_t off_m,
                             uint64_t lo, const uint32_t* qlist, uint32_t* pid, uint32_t* pcnt) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= m) return;
  const uint64_t o = (uint64_t)v * P + part;
  const uint32_t c = pcnt[o], gq = qlist[v];
  uint32_t w = 0;
  for (uint32_t e = 0; e < c; ++e) {
    const uint32_t id = (uint32_t)(pid[o * KP + e] - off_m + lo);
    if (id != gq) pid[o * KP + w++] = id;
  }
  pcnt[o] = w;
}

// Exact global kNN (over all n points, self excluded) of the m query points
// qlist_d[0..m): out_ids_d[v * k ..] = the k smallest (reference fp64
// distance, id) keys of point qlist_d[v], in that order (metrics.hpp:77-91
// exact_knn_ids before its final id sort). FFMA certified filter over the
// whole dataset -> fp64 re-rank -> exhaustive fp64 for uncertified slots.
void knn_global_sample(nomad_b200_ctx* ctx, XPtr x, uint64_t n, uint64_t d,
                       const uint32_t* qlist_d, uint32_t m, uint32_t k, uint32_t* out_ids_d) {
  cudaStream_t S = ctx->stream;
  if (k < 1) fail(kParameter, "k must be >= 1");
  if (k >= n) fail(kParameter, "k must be < n");
  if (m == 0) return;
  if (k > 56) return knn_exhaustive_rows(ctx, x, n, d, qlist_d, m, k, out_ids_d);
  const uint32_t KP = k <= 24 ? 32 : 64;
  // candidates split into P partitions so that the grid covers the GPU
  const uint32_t nt = (m + QT - 1) / QT;
  uint32_t P = 1;
  if (x.bf) {
    P = KP == 32 ? 32 : 16;  // widened chunk by chunk: the most partitions the merge takes
    while (P > 1 && n / P < (uint64_t)CT) P /= 2;
  } else {
    while (P < 16 && nt * P < 2 * (uint32_t)ctx->sm_count && n / (2 * P) >= (uint64_t)CT) P *= 2;
  }
  DBuf<uint32_t> pid((uint64_t)m * P * KP), pcnt((uint64_t)m * P);
  DBuf<float> plb((uint64_t)m * P);
  if (!x.bf) {
    std::vector<FilterSeg> sg;
    for (uint32_t p = 0; p < P; ++p) {
      const uint64_t lo = n * p / P, hi = n * (p + 1) / P;
      sg.push_back(FilterSeg{lo, 0, (uint32_t)(hi - lo), m, nt * p, p});
    }
    ffma_filter(ctx, static_cast<const float*>(x.p), d, nullptr, qlist_d, sg, nt * P, (int)KP,
                (int)P, pid.p, plb.p, pcnt.p);
  } else {
    // bf16 rows: the queries and a chunk of partitions at a time are widened
    // into an f32 scratch [queries | chunk] (<= ~8 GB), filtered, and the
    // chunk's partition lists remapped to global ids
    uint32_t per = P;  // partitions per chunk
    while (per > 1 && (n / P * per + m) * d * 4 > (8ull << 30)) per /= 2;
    const uint64_t max_rows = (n + P - 1) / P * per + per;
    DBuf<float> scr((m + max_rows) * d);
    DBuf<uint32_t> qid(m);
    {
      std::vector<uint32_t> h(m);
      for (uint32_t i = 0; i < m; ++i) h[i] = i;
      NB_CUDA(cudaMemcpyAsync(qid.p, h.data(), m * 4, cudaMemcpyHostToDevice, S));
    }
    k_widen_rows<<<ctx->sm_count * 8, 256, 0, S>>>(x, qlist_d, 0, m, (uint32_t)d, scr.p);
    note_launch(ctx, "k_widen_rows");
    for (uint32_t p0 = 0; p0 < P; p0 += per) {
      const uint64_t clo = n * p0 / P, chi = n * (p0 + per) / P;
      k_widen_rows<<<ctx->sm_count * 8, 256, 0, S>>>(x, nullptr, clo, chi - clo, (uint32_t)d,
                                                     scr.p + (uint64_t)m * d);
      note_launch(ctx, "k_widen_rows");
      std::vector<FilterSeg> sg;
      for (uint32_t p = p0; p < p0 + per; ++p) {
        const uint64_t lo = n * p / P, hi = n * (p + 1) / P;
        sg.push_back(FilterSeg{m + (lo - clo), 0, (uint32_t)(hi - lo), m, nt * (p - p0), p});
      }
      ffma_filter(ctx, scr.p, d, nullptr, qid.p, sg, nt * per, (int)KP, (int)P, pid.p, plb.p,
                  pcnt.p);
      for (uint32_t p = p0; p < p0 + per; ++p) {
        k_remap_part<<<(m + 127) / 128, 128, 0, S>>>(m, P, KP, p, m, clo, qlist_d, pid.p, pcnt.p);
        note_launch(ctx, "k_remap_part");
      }
    }
  }
  const uint32_t KPP = P * KP;
  DBuf<uint32_t> cid((uint64_t)m * KPP), ccnt(m), fb(m), nfb(1);
  DBuf<float> clb(m);
  const unsigned rb = (unsigned)(((uint64_t)m * 32 + 255) / 256);
  k_merge_parts<<<rb, 256, 0, S>>>(m, P, KP, pid.p, plb.p, pcnt.p, cid.p, clb.p, ccnt.p);
  note_launch(ctx, "k_merge_parts");
  NB_CUDA(cudaMemsetAsync(nfb.p, 0, 4, S));
  auto go = [&](auto kp) {
    launch_rerank<decltype(kp)::value>((uint64_t)m, S, x, (uint32_t)d, (uint64_t)m, qlist_d,
                                       (const uint32_t*)nullptr, (const uint32_t*)nullptr, k, k,
                                       (const uint32_t*)cid.p, (const float*)clb.p,
                                       (const uint32_t*)ccnt.p, (const uint32_t*)nullptr,
                                       out_ids_d, (double*)nullptr, fb.p, nfb.p, 1.0, 0);
  };
  switch (KPP) {
    case 32: go(std::integral_constant<int, 32>{}); break;
    case 64: go(std::integral_constant<int, 64>{}); break;
    case 128: go(std::integral_constant<int, 128>{}); break;
    case 256: go(std::integral_constant<int, 256>{}); break;
    case 512: go(std::integral_constant<int, 512>{}); break;
    default: go(std::integral_constant<int, 1024>{}); break;
  }
  note_launch(ctx, "k_knn_rerank");
  uint32_t nf = 0;
  NB_CUDA(cudaMemcpyAsync(&nf, nfb.p, 4, cudaMemcpyDeviceToHost, S));
  NB_CUDA(cudaStreamSynchronize(S));
  if (nf) {
    k_knn_exhaustive<<<nf, 128, 0, S>>>(x, (uint32_t)d, n, qlist_d, nullptr, nullptr, nullptr,
                                        nullptr, k, k, fb.p, nullptr, out_ids_d, nullptr);
    note_launch(ctx, "k_knn_exhaustive");
  }
  NB_CUDA(cudaStreamSynchronize(S));
}

}  // namespace nb

using namespace nb;

extern "C" {

static int32_t build_knn_impl(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                              const nomad_b200_clusters* clusters, uint64_t k, int32_t knn_mode,
                              uint64_t n_owned, const uint32_t* owned, nomad_b200_graph* out) {
  return guard([&] {
    if (!ctx || !clusters || !out) fail(kParameter, "NULL argument");
    if (k < 1) fail(kParameter, "k must be >= 1");
    bind_device(ctx);
    cudaStream_t S = ctx->stream;
    DevData dd;
    dd.bind(data, ctx);
    if (clusters->rows != dd.n) fail(kParameter, "clusters and dataset cover different points");
    if (!clusters->assignment) fail(kParameter, "assignment is NULL");
    const uint32_t C = (uint32_t)clusters->n_clusters;
    DBuf<uint32_t> a_own;
    const uint32_t* a = clusters->assignment;
    if (clusters->location != NOMAD_B200_DEVICE) {
      a_own.alloc(dd.n);
      copy_h2d(ctx, a_own.p, a, dd.n * 4);
      a = a_own.p;
    }
    if (knn_mode != NOMAD_B200_KNN_EXACT && knn_mode != NOMAD_B200_KNN_BF16 &&
        knn_mode != NOMAD_B200_KNN_EXACT_FFMA)
      fail(kParameter, "unknown knn_mode");
    std::vector<uint8_t> own;
    if (owned) {
      own.assign(C, 0);
      for (uint64_t i = 0; i < n_owned; ++i) {
        if (owned[i] >= C) fail(kParameter, "owned cluster id out of range");
        own[owned[i]] = 1;
      }
    }
    const bool dbg = std::getenv("NOMAD_B200_DEBUG_KNN") != nullptr;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](const char* what) {
      if (!dbg) return;
      NB_CUDA(cudaStreamSynchronize(S));
      const auto now = std::chrono::steady_clock::now();
      std::fprintf(stderr, "knn call  %-28s %8.1f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - t0).count());
      t0 = now;
    };
    lap("inputs");
    KnnResult R;
    build_knn_exact(ctx, dd.x, dd.n, dd.d, a, C, (uint32_t)k, R, knn_mode, owned ? &own : nullptr);
    lap("build");
    ctx->knn_tc_uncertified = R.tc_uncertified;
    ctx->knn_sub_certified = R.sub_certified;
    ctx->knn_exhaustive = R.fallbacks;
    const bool dev = out->location == NOMAD_B200_DEVICE;
    copy_out(ctx, out->offsets, R.offsets.p, (dd.n + 1) * 4, dev);
    if (R.edges) {
      copy_out(ctx, out->neighbors, R.nb.p, R.edges * 4, dev);
      if (out->distances) copy_out(ctx, out->distances, R.dist.p, R.edges * 8, dev);
    }
    lap("outputs");
    out->rows = dd.n;
    out->k = k;
  });
}

int32_t nomad_b200_build_knn(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                             const nomad_b200_clusters* clusters, uint64_t k, int32_t knn_mode,
                             nomad_b200_graph* out) {
  return build_knn_impl(ctx, data, clusters, k, knn_mode, 0, nullptr, out);
}

int32_t nomad_b200_build_knn_shard(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                   const nomad_b200_clusters* clusters, uint64_t k,
                                   int32_t knn_mode, uint64_t n_owned,
                                   const uint32_t* owned_clusters, nomad_b200_graph* out) {
  if (!owned_clusters && n_owned) return guard([&] { fail(kParameter, "owned_clusters is NULL"); });
  static const uint32_t none = 0;
  return build_knn_impl(ctx, data, clusters, k, knn_mode, n_owned,
                        owned_clusters ? owned_clusters : &none, out);
}

// recall@k of a graph against the exact lists of `sample` rows drawn without
// replacement (splitmix order), each recomputed exhaustively in fp64.
int32_t nomad_b200_knn_recall(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                              const nomad_b200_clusters* clusters,
                              const nomad_b200_graph* graph, uint64_t sample, uint64_t seed,
                              double* recall_out) {
  return guard([&] {
    if (!ctx || !clusters || !graph || !recall_out) fail(kParameter, "NULL argument");
    bind_device(ctx);
    cudaStream_t S = ctx->stream;
    DevData dd;
    dd.bind(data, ctx);
    const uint64_t n = dd.n, k = graph->k;
    const uint32_t C = (uint32_t)clusters->n_clusters;
    if (graph->rows != n || clusters->rows != n) fail(kParameter, "row counts differ");
    std::vector<uint32_t> a(n), off(n + 1);
    const auto kind_a = clusters->location == NOMAD_B200_DEVICE ? cudaMemcpyDeviceToHost
                                                                : cudaMemcpyHostToHost;
    const auto kind_g = graph->location == NOMAD_B200_DEVICE ? cudaMemcpyDeviceToHost
                                                             : cudaMemcpyHostToHost;
    NB_CUDA(cudaMemcpy(a.data(), clusters->assignment, n * 4, kind_a));
    NB_CUDA(cudaMemcpy(off.data(), graph->offsets, (n + 1) * 4, kind_g));
    std::vector<uint32_t> nbh(off[n]);
    if (off[n]) NB_CUDA(cudaMemcpy(nbh.data(), graph->neighbors, (size_t)off[n] * 4, kind_g));
    // sample rows with a non-empty list
    std::vector<uint32_t> rows;
    {
      std::vector<uint32_t> cand;
      for (uint64_t i = 0; i < n; ++i)
        if (off[i + 1] > off[i]) cand.push_back((uint32_t)i);
      uint64_t st = seed ^ 0x7265636c6c21ull;
      const uint64_t m = std::min<uint64_t>(sample ? sample : cand.size(), cand.size());
      for (uint64_t t = 0; t < m; ++t) {  // partial Fisher-Yates
        st += 0x9E3779B97F4A7C15ull;
        uint64_t z = st;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const uint64_t j = t + z % (cand.size() - t);
        std::swap(cand[t], cand[j]);
      }
      rows.assign(cand.begin(), cand.begin() + m);
    }
    if (rows.empty()) {
      *recall_out = 1.0;
      return;
    }
    DBuf<uint32_t> a_d(n), sizes(C), mem, rows_d(rows.size()), off_d(n + 1), nb2(off[n] + 1);
    NB_CUDA(cudaMemcpyAsync(a_d.p, a.data(), n * 4, cudaMemcpyHostToDevice, S));
    NB_CUDA(cudaMemcpyAsync(off_d.p, off.data(), (n + 1) * 4, cudaMemcpyHostToDevice, S));
    NB_CUDA(cudaMemcpyAsync(rows_d.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice, S));
    NB_CUDA(cudaMemsetAsync(sizes.p, 0, C * 4, S));
    k_sizes2<<<(unsigned)std::min<uint64_t>(4096, (n + 255) / 256), 256, 0, S>>>(a_d.p, n, sizes.p);
    note_launch(ctx, "k_sizes");
    std::vector<uint64_t> coff;
    group_by_label(ctx, a_d.p, n, C, mem, coff);
    std::vector<uint64_t> cb(coff.begin(), coff.end() - 1);
    DBuf<uint64_t> cb_d(C);
    NB_CUDA(cudaMemcpyAsync(cb_d.p, cb.data(), C * 8, cudaMemcpyHostToDevice, S));
    k_knn_exhaustive<<<(unsigned)rows.size(), 128, 0, S>>>(dd.x, (uint32_t)dd.d, n, nullptr, a_d.p,
                                                          mem.p, cb_d.p, sizes.p, (uint32_t)k, 0u,
                                                          rows_d.p, off_d.p, nb2.p, nullptr);
    note_launch(ctx, "k_knn_exhaustive");
    std::vector<uint32_t> ex(off[n]);
    NB_CUDA(cudaMemcpyAsync(ex.data(), nb2.p, (size_t)off[n] * 4, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    uint64_t hits = 0, total = 0;
    for (uint32_t q : rows) {
      std::vector<uint32_t> e(ex.begin() + off[q], ex.begin() + off[q + 1]);
      std::sort(e.begin(), e.end());
      for (uint32_t t = off[q]; t < off[q + 1]; ++t)
        hits += std::binary_search(e.begin(), e.end(), nbh[t]) ? 1 : 0;
      total += off[q + 1] - off[q];
    }
    *recall_out = total ? (double)hits / (double)total : 1.0;
  });
}

int32_t nomad_b200_knn_stats(nomad_b200_ctx* ctx, uint64_t* tc_uncertified,
                             uint64_t* exhaustive_rows) {
  return guard([&] {
    if (!ctx) fail(kParameter, "NULL argument");
    if (tc_uncertified) *tc_uncertified = ctx->knn_tc_uncertified;
    if (exhaustive_rows) *exhaustive_rows = ctx->knn_exhaustive;
  });
}

int32_t nomad_b200_knn_subcluster_rows(nomad_b200_ctx* ctx, uint64_t* rows) {
  return guard([&] {
    if (!ctx || !rows) fail(kParameter, "NULL argument");
    *rows = ctx->knn_sub_certified;
  });
}

}  // extern "C"
