// kNN distance filter on the 5th-gen tensor cores (knn.hpp:65-109).
//
// Per cluster, rows are centred on the cluster mean (u = x - mu, fp64) and
// rounded to 16 bits into a padded cluster-contiguous copy; every (query
// tile, candidate tile) product S = U_q U_c^T (128 x 256, K = d) runs on
// tcgen05.mma with operands streamed by TMA into 128B-swizzled shared memory
// (4-stage ring) and the fp32 accumulator double-buffered in TMEM. Warp 0
// issues TMA, warp 1 issues MMAs, warps 2-5 run the epilogue (tcgen05.ld, one
// query row per thread, distance ||u_q||^2 + ||u_c||^2 - 2 S, register-
// resident sorted top-KP with rolled insertion).
//
// Two uses:
//  * fast mode (NOMAD_B200_KNN_BF16): bf16 operands, KP = 32 survivors,
//    re-ranked in exact fp64 (knn.cu) — recall@k vs the exact mode is reported.
//  * certified exact mode: fp16 operands (11-bit mantissa), KP = 64 survivors
//    and a rigorous lower bound on the reference distance of every excluded
//    candidate; the re-rank certifies the top-k or sends the row to the
//    exhaustive fp64 fallback, so ids and distances are bit-identical to the
//    reference.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "index_common.cuh"
#include "tc_common.cuh"

namespace nb {

namespace {

constexpr int TM = 128;       // query rows per CTA (UMMA M)
constexpr int TN = 128;       // tile width of the diagnostic GEMM
constexpr int TN2 = 256;      // candidate rows per tile (UMMA N)
constexpr int KC = 64;        // 16-bit columns per stage (one 128B swizzle atom)
constexpr int STAGES2 = 4;
constexpr int QCAP = 16;     // per-thread queue of below-threshold hits (epilogue)
#ifndef TC_EXP
#define TC_EXP 0
#endif
constexpr uint32_t STAGE_BYTES = (TM + TN) * KC * 2;    // diagnostic GEMM
constexpr uint32_t STAGE2_BYTES = (TM + TN2) * KC * 2;  // 48 KB

struct TcTile {
  uint32_t row0;   // padded row of this query tile
  uint32_t cbase;  // padded row of the cluster's first member
  uint32_t size;   // cluster size
  uint32_t qoff;   // query offset inside the cluster
  uint32_t cid;    // cluster id
};

// Error model of the certified filter (scaled units, see the host side):
//   g_acc    relative error of S and of the norms: tcgen05 fp32 accumulation
//            (taken as <= 2 ulp per addition over dpad additions), the fp32
//            norm chains and the two final fp32 roundings, x1.5
//   eps      componentwise relative rounding of u to fp16 (fp64 -> fp32 -> fp16)
//   abs_norm fp16 subnormal absolute rounding, 2^-25 sqrt(dpad)
struct CertParams {
  float g_acc;
  float eps;
  float abs_norm;
  float inv_s2;  // 1 / scale^2
  float g64;     // reference fp64 chain relative error (2 (d + 1) u64)
};

template <bool FP16>
__device__ __forceinline__ uint16_t to16(float v) {
  if constexpr (FP16) return __half_as_ushort(__float2half_rn(v));
  else return __bfloat16_as_ushort(__float2bfloat16_rn(v));
}
template <bool FP16>
__device__ __forceinline__ float from16(uint16_t b) {
  if constexpr (FP16) return __half2float(__ushort_as_half(b));
  else return __bfloat162float(__ushort_as_bfloat16(b));
}

__global__ void k_tc_absmax(XPtr x, uint64_t d, const uint32_t* perm_pad,
                            const uint32_t* row_cl, const double* means, uint64_t rows_pad,
                            unsigned int* amax_bits) {
  const uint64_t row = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows_pad) return;
  const uint32_t id = perm_pad[row];
  if (id == 0xFFFFFFFFu) return;
  const double* mu = means + (uint64_t)row_cl[row] * d;
  float m = 0.f;
  for (uint64_t j = lane; j < d; j += 32)
    m = fmaxf(m, fabsf((float)((double)x[(uint64_t)id * d + j] - mu[j])));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) atomicMax(amax_bits, __float_as_uint(m));
}

// 16-bit (scale * (x - mu)) into the padded copy; fp32 norms of the rounded rows.
template <bool FP16>
__global__ void k_tc_prep(XPtr x, uint64_t d, uint64_t dpad,
                          const uint32_t* __restrict__ perm_pad, const uint32_t* __restrict__ row_cl,
                          const double* __restrict__ means, uint64_t rows_pad, float scale,
                          uint16_t* __restrict__ xb, float* __restrict__ norms) {
  const uint64_t row = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows_pad) return;
  const uint32_t id = perm_pad[row];
  const double* mu = means + (uint64_t)row_cl[row] * d;
  float acc = 0.f;
  for (uint64_t j = lane; j < dpad; j += 32) {
    float v = 0.f;
    if (id != 0xFFFFFFFFu && j < d) v = (float)((double)x[(uint64_t)id * d + j] - mu[j]) * scale;
    const uint16_t b = to16<FP16>(v);
    xb[row * dpad + j] = b;
    const float bf = from16<FP16>(b);
    acc = fmaf(bf, bf, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) norms[row] = acc;
}

template <int KP, bool CERT>
__global__ void __launch_bounds__(192, 1) k_knn_tc2(const __grid_constant__ CUtensorMap tmap,
                                                    const TcTile* __restrict__ tiles,
                                                    const float* __restrict__ norms,
                                                    const float* __restrict__ cl_maxnorm,
                                                    const uint32_t* __restrict__ perm_pad,
                                                    uint32_t kchunks, uint32_t idesc,
                                                    CertParams cp, uint32_t* cand_ids,
                                                    float* cand_lb, uint32_t* cand_cnt) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = smem + ((1024 - (tc::smem_u32(smem) & 1023)) & 1023);
  uint8_t* stage_mem = base;
  float* cn = reinterpret_cast<float*>(base + STAGES2 * STAGE2_BYTES);  // 2 x TN2 norms
  uint64_t* full = reinterpret_cast<uint64_t*>(cn + 2 * TN2);
  uint64_t* empty = full + STAGES2;
  uint64_t* tfull = empty + STAGES2;  // 2
  uint64_t* tempty = tfull + 2;       // 2
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* spill = reinterpret_cast<float*>(tmem_slot + 4);  // 128 x 33 (epilogue scratch)

  const TcTile T = tiles[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 1) tc::tmem_alloc(tmem_slot, 2 * TN2);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 128);
    }
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t ntiles = (T.size + TN2 - 1) / TN2;
  const uint32_t total = ntiles * kchunks;

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer
      for (uint32_t it = 0; it < total; ++it) {
        const uint32_t s = it % STAGES2;
        if (it >= STAGES2) tc::mbar_wait(&empty[s], ((it / STAGES2) - 1) & 1);
        const uint32_t ct = it / kchunks, kc = it % kchunks;
        uint8_t* sa = stage_mem + s * STAGE2_BYTES;
#if TC_EXP == 2  // timing experiment: no operand traffic after the first fill
        if (it >= STAGES2) { tc::mbar_arrive(&full[s]); continue; }
#endif
        tc::mbar_expect_tx(&full[s], STAGE2_BYTES);
        tc::tma_load_2d(sa, &tmap, &full[s], (int32_t)(kc * KC), (int32_t)T.row0);
        tc::tma_load_2d(sa + TM * KC * 2, &tmap, &full[s], (int32_t)(kc * KC),
                        (int32_t)(T.cbase + ct * TN2));
        tc::tma_load_2d(sa + (TM + 128) * KC * 2, &tmap, &full[s], (int32_t)(kc * KC),
                        (int32_t)(T.cbase + ct * TN2 + 128));
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer
      for (uint32_t ct = 0; ct < ntiles; ++ct) {
        const uint32_t b = ct & 1;
        if (ct >= 2) tc::mbar_wait(&tempty[b], ((ct >> 1) - 1) & 1);
        tc::fence_after();
        const uint32_t acc = tmem + b * TN2;
        for (uint32_t kc = 0; kc < kchunks; ++kc) {
          const uint32_t it = ct * kchunks + kc, s = it % STAGES2;
          tc::mbar_wait(&full[s], (it / STAGES2) & 1);
          tc::fence_after();
          const uint32_t sa = tc::smem_u32(stage_mem + s * STAGE2_BYTES);
          const uint64_t da = tc::sdesc_k_sw128(sa), db = tc::sdesc_k_sw128(sa + TM * KC * 2);
#pragma unroll
          for (int k = 0; k < KC / 16; ++k)
            tc::umma_bf16(acc, da + 2 * k, db + 2 * k, idesc, (kc | k) != 0);
          tc::umma_commit(&empty[s]);
        }
        tc::umma_commit(&tfull[b]);
      }
    }
  } else {
    // ---- epilogue: row r <-> TMEM lane r
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..127
    const uint32_t q_local = T.qoff + r;
    const bool qvalid = q_local < T.size;
    const float qn = norms[T.row0 + r];
    float ld[KP];
    uint32_t li[KP];
#pragma unroll
    for (int e = 0; e < KP; ++e) {
      ld[e] = __int_as_float(0x7f800000);
      li[e] = 0xFFFFFFFFu;
    }
    float tau = ld[KP - 1];
    float* qd = spill + 128 * 33;  // hit queue, [QCAP][128] (conflict-free)
    uint8_t* qc = reinterpret_cast<uint8_t*>(qd + QCAP * 128);
    uint32_t qn_cnt = 0, qtile = 0;
    // insert the queued hits of tile qtile in column order (strict <, so the
    // list equals immediate insertion)
    auto flush = [&]() {
      for (uint32_t i = 0; i < qn_cnt; ++i) {
        float cd = qd[i * 128 + et];
        if (!(cd < tau)) continue;
        uint32_t ci = qtile * TN2 + qc[i * 128 + et];
#pragma unroll
        for (int e = 0; e < KP; ++e) {
          if (cd < ld[e]) {
            const float td = ld[e];
            const uint32_t ti = li[e];
            ld[e] = cd;
            li[e] = ci;
            cd = td;
            ci = ti;
          }
        }
        tau = ld[KP - 1];
      }
      qn_cnt = 0;
    };
    // candidate norms (invalid -> +inf), loaded one tile ahead
    constexpr int NPT = TN2 / 128;
    float nx[NPT];
    auto load_norms = [&](uint32_t ct) {
#pragma unroll
      for (int i = 0; i < NPT; ++i) {
        const uint32_t cl = ct * TN2 + et + 128 * i;
        nx[i] = cl < T.size ? __ldg(norms + T.cbase + cl) : __int_as_float(0x7f800000);
      }
    };
    load_norms(0);
    for (uint32_t ct = 0; ct < ntiles; ++ct) {
      const uint32_t b = ct & 1;
      qtile = ct;
      float* cnb = cn + b * TN2;
#pragma unroll
      for (int i = 0; i < NPT; ++i) cnb[et + 128 * i] = nx[i];
      if (ct + 1 < ntiles) load_norms(ct + 1);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tc::mbar_wait(&tfull[b], (ct >> 1) & 1);
      tc::fence_after();
      const uint32_t acc = tmem + b * TN2 + ((uint32_t)(q4 * 32) << 16);
#pragma unroll 1
      for (int cc = 0; cc < TN2; cc += 32) {
        float v[32];
        tc::tmem_ld32(acc + cc, v);
#if TC_EXP == 1  // timing experiment: epilogue only drains TMEM
        continue;
#endif
        if (!qvalid) continue;
        // distances (straight-line), then the below-threshold hits
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = fmaf(-2.f, v[j], qn + cnb[cc + j]);
        // common case: nothing in these 32 columns beats tau (min tree);
        // the query's own column always does, once per query
        float t[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) t[j] = fminf(v[j], v[j + 16]);
#pragma unroll
        for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
          for (int j = 0; j < w; ++j) t[j] = fminf(t[j], t[j + w]);
        if (!(t[0] < tau)) continue;
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) mask |= (v[j] < tau ? 1u : 0u) << j;
        // the query itself is never a candidate
        const uint32_t self = q_local - (ct * TN2 + cc);
        if (self < 32) mask &= ~(1u << self);
        if (mask) {
          // queue this chunk's hits (column offset in the tile as u8); the
          // list insertions run once per tile, so a warp pays for the lane
          // with the most hits in the tile rather than in every chunk
          float* row = spill + et * 33;
#pragma unroll
          for (int j = 0; j < 32; ++j) row[j] = v[j];
          while (mask) {
            if (qn_cnt == QCAP) flush();
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            qd[qn_cnt * 128 + et] = row[j];
            qc[qn_cnt * 128 + et] = (uint8_t)(cc + j);
            ++qn_cnt;
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&tempty[b]);  // TMEM drained; hits are in the queue
      flush();
    }
    if (qvalid) {
      const uint32_t gq = perm_pad[T.row0 + r];
      uint32_t c = 0;
#pragma unroll
      for (int e = 0; e < KP; ++e)
        if (li[e] != 0xFFFFFFFFu) {
          cand_ids[(uint64_t)gq * KP + c] = perm_pad[T.cbase + li[e]];
          ++c;
        }
      cand_cnt[gq] = c;
      float lb = __int_as_float(0x7f800000);  // complete list: nothing excluded
      if (CERT && c == KP) {
        // Every excluded candidate j has Dtilde_j >= T = tau (scaled units).
        // With a = ||u_b,q||, s = ||u_b,q - u_b,j|| and ||u_b,j|| <= a + s:
        //   T <= Dtilde_j <= s^2 + g (2a + s)^2
        //   => s >= (-2ga + sqrt(4g^2a^2 + (1+g)(T - 4ga^2))) / (1+g)
        // The rounding to 16 bits moves each vector by <= eps ||u|| + abs:
        //   t = ||u_q - u_j|| >= (s - 2 eps a_true - 2 abs) / (1 + eps)
        //   ref_j >= t^2 (1 - g64) / scale^2
        // (double precision, rounded down at the end; no cluster-wide norm)
        const double g = cp.g_acc, a = sqrt((double)qn) * (1.0 + 1e-6);
        const double disc = 4.0 * g * g * a * a + (1.0 + g) * ((double)tau - 4.0 * g * a * a);
        const double s = fmax((-2.0 * g * a + sqrt(fmax(disc, 0.0))) / (1.0 + g), 0.0);
        const double eps = cp.eps, a_true = a / (1.0 - eps) + cp.abs_norm;
        const double t = fmax((s - 2.0 * eps * a_true - 2.0 * cp.abs_norm) / (1.0 + eps), 0.0);
        lb = __double2float_rd(t * t * cp.inv_s2 * (1.0 - cp.g64) * (1.0 - 1e-9));
      }
      cand_lb[gq] = lb;
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 2 * TN2);
}

// Debug / unit path: D = A B^T for one 128 x 128 tile pair (rows a0, b0 of
// the 16-bit tensor), written to out[128][128].
__global__ void __launch_bounds__(128, 1) k_tc_gemm_tile(const __grid_constant__ CUtensorMap tmap,
                                                         uint32_t a0, uint32_t b0,
                                                         uint32_t kchunks, uint32_t idesc,
                                                         float* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = smem + ((1024 - (tc::smem_u32(smem) & 1023)) & 1023);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + STAGE_BYTES);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);
  const int r = threadIdx.x, warp = r >> 5;
  if (warp == 0) tc::tmem_alloc(tmem_slot, TN);
  if (r == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
  if (r == 0) {
    for (uint32_t kc = 0; kc < kchunks; ++kc) {
      tc::mbar_expect_tx(&bar[0], STAGE_BYTES);
      tc::tma_load_2d(base, &tmap, &bar[0], (int32_t)(kc * KC), (int32_t)a0);
      tc::tma_load_2d(base + TM * KC * 2, &tmap, &bar[0], (int32_t)(kc * KC), (int32_t)b0);
      tc::mbar_wait(&bar[0], kc & 1);
      tc::fence_after();
      const uint32_t sa = tc::smem_u32(base);
      const uint64_t da = tc::sdesc_k_sw128(sa), db = tc::sdesc_k_sw128(sa + TM * KC * 2);
      for (int k = 0; k < KC / 16; ++k)
        tc::umma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (kc | k) != 0);
      tc::umma_commit(&bar[1]);
      tc::mbar_wait(&bar[1], kc & 1);
    }
  }
  __syncwarp();
  __syncthreads();
  tc::fence_after();
  for (int cc = 0; cc < TN; cc += 32) {
    float v[32];
    tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + cc, v);
    for (int j = 0; j < 32; ++j) out[r * TN + cc + j] = v[j];
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, TN);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    NB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) fail(kInternal, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

CUtensorMap make_tmap(const uint16_t* xb, uint64_t rows, uint64_t dpad, bool fp16) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  const cuuint64_t gdim[2] = {dpad, rows};
  const cuuint64_t gstride[1] = {dpad * 2};
  const cuuint32_t box[2] = {KC, TM};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(
      &m, fp16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)xb,
      gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(kInternal, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}

// kind::f16 instruction descriptor: fp32 D, A/B = bf16 (1) or fp16 (0).
constexpr uint32_t idesc16(uint32_t M, uint32_t N, bool fp16) {
  return (1u << 4) | ((fp16 ? 0u : 1u) << 7) | ((fp16 ? 0u : 1u) << 10) | ((N >> 3) << 17) |
         ((M >> 4) << 24);
}

}  // namespace

// Candidate generation on the tensor cores. fp16 == certified exact filter
// (KP = 64, cand_lb = rigorous lower bound on excluded reference distances);
// otherwise the bf16 fast filter (KP = 32, cand_lb = +inf).
// NOMAD_B200_DEBUG_KNN=2: per-step timing of the tensor-core stage
static void tc_lap(cudaStream_t S, const char* what) {
  static const bool on = [] {
    const char* e = std::getenv("NOMAD_B200_DEBUG_KNN");
    return e && std::atoi(e) >= 2;
  }();
  if (!on) return;
  static auto t_last = std::chrono::steady_clock::now();
  NB_CUDA(cudaStreamSynchronize(S));
  const auto now = std::chrono::steady_clock::now();
  std::fprintf(stderr, "      tc %-20s %7.1f ms\n", what,
               std::chrono::duration<double, std::milli>(now - t_last).count());
  t_last = now;
}

// Padded cluster-contiguous layout of one group: row p of cluster slot g
// (padded start gl[3g]) holds member p - gl[3g] (or no row: padding);
// rcl[p] = that cluster's id. Rows past the last slot belong to slot 0.
__global__ void k_tc_layout(const uint32_t* __restrict__ mem, const uint32_t* __restrict__ grp,
                            const uint64_t* __restrict__ gl, uint32_t G, uint64_t rows,
                            uint32_t* perm, uint32_t* rcl) {
  const uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (p >= rows) return;
  uint32_t lo = 0, hi = G;  // last slot with start <= p
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (gl[3 * mid] <= p) lo = mid; else hi = mid;
  }
  const uint64_t t = p - gl[3 * lo];
  const bool in = gl[3 * lo] <= p && t < gl[3 * lo + 2];
  perm[p] = in ? mem[gl[3 * lo + 1] + t] : 0xFFFFFFFFu;
  rcl[p] = grp[lo];
}

// cmax[c] = max over the cluster's padded rows of sqrt(norm) * 1.0001 (the
// float bits of non-negative values order like unsigned integers)
__global__ void k_tc_cmax(const float* __restrict__ norms, const uint32_t* __restrict__ rcl,
                          uint64_t rows, unsigned* cmax) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= rows) return;
  atomicMax(cmax + rcl[i], __float_as_uint(sqrtf(norms[i]) * 1.0001f));
}

// One group of clusters: the padded cluster-contiguous 16-bit copy (tiles
// never straddle a cluster start), its norms and scale, and the candidate
// kernel; candidates land at the rows' global ids.
static void tc_group(nomad_b200_ctx* ctx, XPtr x, uint64_t d, uint64_t dpad, bool fp16, int KP,
                     uint32_t C,
                     const std::vector<uint64_t>& off, const uint32_t* mem_d,
                     const std::vector<uint32_t>& grp, const double* means_p,
                     DBuf<uint32_t>& cand_ids, DBuf<float>& cand_lb, DBuf<uint32_t>& cand_cnt,
                     uint32_t max_qtiles) {
  cudaStream_t S = ctx->stream;
  const uint32_t G = (uint32_t)grp.size();
  std::vector<uint64_t> pstart(G + 1, 0);
  for (uint32_t g = 0; g < G; ++g)
    pstart[g + 1] = pstart[g] + (off[grp[g] + 1] - off[grp[g]] + TM - 1) / TM * TM;
  const uint64_t rows_pad = std::max<uint64_t>(pstart[G], TM);
  if (rows_pad >= (1ull << 31)) fail(kSize, "tensor-core kNN: too many rows for TMA coordinates");
  // rcl: the row's cluster id (means, certificate); tiles carry the group-local cluster index
  std::vector<TcTile> tiles;
  std::vector<uint64_t> gl(3 * (size_t)G);  // per group cluster: padded start, member offset, size
  for (uint32_t g = 0; g < G; ++g) {
    const uint32_t r = grp[g];
    const uint64_t sz = off[r + 1] - off[r];
    gl[3 * g] = pstart[g];
    gl[3 * g + 1] = off[r];
    gl[3 * g + 2] = sz;
    for (uint64_t q = 0; q < sz && (max_qtiles == 0 || q < (uint64_t)max_qtiles * TM); q += TM)
      tiles.push_back(TcTile{(uint32_t)(pstart[g] + q), (uint32_t)pstart[g], (uint32_t)sz,
                             (uint32_t)q, r});
  }
  DBuf<uint32_t> perm_d(rows_pad), rcl_d(rows_pad), grp_d(G);
  DBuf<uint64_t> gl_d(3 * (size_t)G);
  NB_CUDA(cudaMemcpyAsync(grp_d.p, grp.data(), G * 4, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(gl_d.p, gl.data(), gl.size() * 8, cudaMemcpyHostToDevice, S));
  k_tc_layout<<<(unsigned)((rows_pad + 255) / 256), 256, 0, S>>>(mem_d, grp_d.p, gl_d.p, G,
                                                                 rows_pad, perm_d.p, rcl_d.p);
  note_launch(ctx, "k_tc_layout");
  tc_lap(S, "layout");
  // power-of-two scale keeping |u| well inside the 16-bit range
  DBuf<unsigned int> amax(1);
  NB_CUDA(cudaMemsetAsync(amax.p, 0, 4, S));
  const unsigned rb = (unsigned)((rows_pad * 32 + 255) / 256);
  k_tc_absmax<<<rb, 256, 0, S>>>(x, d, perm_d.p, rcl_d.p, means_p, rows_pad, amax.p);
  note_launch(ctx, "k_tc_absmax");
  unsigned int ab = 0;
  NB_CUDA(cudaMemcpyAsync(&ab, amax.p, 4, cudaMemcpyDeviceToHost, S));
  NB_CUDA(cudaStreamSynchronize(S));
  float amx;
  std::memcpy(&amx, &ab, 4);
  float scale = 1.f;
  if (amx > 0.f && std::isfinite(amx)) {
    const float target = 1024.f;  // max |scaled u|: squares and sums stay far from overflow
    scale = std::ldexp(1.f, (int)std::floor(std::log2(target / amx)));
  }
  DBuf<uint16_t> xb(rows_pad * dpad);
  DBuf<float> norms(rows_pad);
  if (fp16)
    k_tc_prep<true><<<rb, 256, 0, S>>>(x, d, dpad, perm_d.p, rcl_d.p, means_p, rows_pad, scale,
                                       xb.p, norms.p);
  else
    k_tc_prep<false><<<rb, 256, 0, S>>>(x, d, dpad, perm_d.p, rcl_d.p, means_p, rows_pad, scale,
                                        xb.p, norms.p);
  note_launch(ctx, "k_tc_prep");
  tc_lap(S, "absmax + prep");
  // per-cluster max ||u_b|| (scaled), for the certificate
  DBuf<float> cmax_d(C);
  NB_CUDA(cudaMemsetAsync(cmax_d.p, 0, C * 4, S));
  k_tc_cmax<<<(unsigned)((rows_pad + 255) / 256), 256, 0, S>>>(norms.p, rcl_d.p, rows_pad,
                                                               reinterpret_cast<unsigned*>(cmax_d.p));
  note_launch(ctx, "k_tc_cmax");

  tc_lap(S, "norms + cmax");
  if (tiles.empty()) return;
  const CUtensorMap tm = make_tmap(xb.p, rows_pad, dpad, fp16);
  DBuf<TcTile> tiles_d(tiles.size());
  NB_CUDA(cudaMemcpyAsync(tiles_d.p, tiles.data(), tiles.size() * sizeof(TcTile),
                          cudaMemcpyHostToDevice, S));
  CertParams cp;
  const double u32 = 0x1p-24;
  cp.g_acc = (float)(((double)dpad * 2.0 * 2 * u32 + (double)(dpad / 32 + 6) * u32 + 4 * u32) *
                     1.5);
  cp.eps = (float)(0x1p-11 + u32 + 1e-12);
  cp.abs_norm = (float)(0x1p-25 * std::sqrt((double)dpad));
  cp.inv_s2 = 1.f / (scale * scale);
  cp.g64 = (float)((double)(d + 1) * 0x1p-53 * 2);
  const size_t smem = 1024 + STAGES2 * STAGE2_BYTES + 2 * TN2 * 4 + (2 * STAGES2 + 4) * 8 + 16 +
                      128 * 33 * 4 + QCAP * 128 * 5;
  auto go = [&](auto kern) {
    NB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)tiles.size(), 192, smem, S>>>(tm, tiles_d.p, norms.p, cmax_d.p, perm_d.p,
                                                   (uint32_t)(dpad / KC), idesc16(TM, TN2, fp16),
                                                   cp, cand_ids.p, cand_lb.p, cand_cnt.p);
  };
  if (fp16 && KP == 64) go(k_knn_tc2<64, true>);
  else if (fp16) go(k_knn_tc2<32, true>);
  else go(k_knn_tc2<32, false>);
  note_launch(ctx, "k_knn_tc2");
  NB_CUDA(cudaStreamSynchronize(S));
  tc_lap(S, "k_knn_tc2");
}

void knn_tc_candidates(nomad_b200_ctx* ctx, XPtr x, uint64_t n, uint64_t d,
                       const uint32_t* assign_d, uint32_t C, bool fp16, DBuf<uint32_t>& cand_ids,
                       DBuf<float>& cand_lb, DBuf<uint32_t>& cand_cnt, int* kp_out,
                       const std::vector<uint8_t>* own, int kp16, uint32_t max_qtiles,
                       bool keep) {
  cudaStream_t S = ctx->stream;
  const int KP = fp16 ? (kp16 == 32 ? 32 : 64) : 32;
  *kp_out = KP;
  DBuf<uint32_t> mem;
  std::vector<uint64_t> off;
  group_by_label(ctx, assign_d, n, C, mem, off);
  // centring vectors: the clusters' means in a fixed parallel summation order
  // (any fixed vector keeps the certificate valid)
  DBuf<double> means((uint64_t)C * d);
  NB_CUDA(cudaMemsetAsync(means.p, 0, (uint64_t)C * d * 8, S));
  {
    std::vector<uint64_t> beg, cnt;
    std::vector<uint32_t> rows;
    for (uint32_t r = 0; r < C; ++r)
      if (off[r + 1] > off[r]) {
        beg.push_back(off[r]);
        cnt.push_back(off[r + 1] - off[r]);
        rows.push_back(r);
      }
    fast_column_means(ctx, x, d, mem.p, beg, cnt, rows, means.p);
  }
  tc_lap(S, "grouping + means");
  if (!keep) {  // (keep: a second pass over other clusters into the same lists)
    cand_ids.alloc(n * (uint64_t)KP);
    cand_lb.alloc(n);
    cand_cnt.alloc(n);
    NB_CUDA(cudaMemsetAsync(cand_cnt.p, 0, n * 4, S));
    // rows no pass reaches keep an empty list with bound 0: never certified
    NB_CUDA(cudaMemsetAsync(cand_lb.p, 0, n * 4, S));
  }
  const uint64_t dpad = (d + KC - 1) / KC * KC;
  // Clusters are processed in groups whose padded 16-bit copy fits half of
  // the free device memory (one group unless the dataset is very large, e.g.
  // 60M x 768 bf16 next to its own 92 GB); only clusters with lists to build
  // (size >= 2, owned) enter the copy.
  uint64_t row_budget;
  {
    size_t fr = 0, tot = 0;
    NB_CUDA(cudaMemGetInfo(&fr, &tot));
    row_budget = std::max<uint64_t>(TM, (uint64_t)(fr / 2) / (dpad * 2 + 16));
    row_budget = std::min<uint64_t>(row_budget, (1ull << 31) - 2 * TM);
    if (const char* e = getenv("NOMAD_B200_TC_ROW_BUDGET"))  // tests: force several groups
      row_budget = std::max<uint64_t>(TM, strtoull(e, nullptr, 10));
  }
  std::vector<uint32_t> todo;
  for (uint32_t r = 0; r < C; ++r)
    if (off[r + 1] - off[r] >= 2 && !(own && !(*own)[r])) todo.push_back(r);
  size_t gi = 0;
  while (gi < todo.size()) {
    // one group: consecutive clusters of `todo` within the row budget
    std::vector<uint32_t> grp;
    uint64_t acc = 0;
    while (gi < todo.size()) {
      const uint32_t r = todo[gi];
      const uint64_t pr = (off[r + 1] - off[r] + TM - 1) / TM * TM;
      if (!grp.empty() && acc + pr > row_budget) break;
      grp.push_back(r);
      acc += pr;
      ++gi;
    }
    tc_group(ctx, x, d, dpad, fp16, KP, C, off, mem.p, grp, means.p, cand_ids, cand_lb, cand_cnt,
             max_qtiles);
  }
}

// Unit check of the tcgen05 path: rows of a (rows x d) f32 host matrix are
// rounded to bf16 / fp16; returns D = A[a0:a0+128] B[b0:b0+128]^T.
void tc_gemm_tile_check(nomad_b200_ctx* ctx, const float* host, uint64_t rows, uint64_t d,
                        uint32_t a0, uint32_t b0, bool fp16, float* out_host) {
  cudaStream_t S = ctx->stream;
  const uint64_t dpad = (d + KC - 1) / KC * KC;
  std::vector<uint16_t> hb(rows * dpad);
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t j = 0; j < dpad; ++j) {
      const float v = j < d ? host[i * d + j] : 0.f;
      hb[i * dpad + j] = fp16 ? __half_as_ushort(__float2half_rn(v))
                              : __bfloat16_as_ushort(__float2bfloat16_rn(v));
    }
  DBuf<uint16_t> xb(rows * dpad);
  NB_CUDA(cudaMemcpy(xb.p, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
  const CUtensorMap tm = make_tmap(xb.p, rows, dpad, fp16);
  DBuf<float> out(TM * TN);
  const size_t smem = 1024 + STAGE_BYTES + 64;
  NB_CUDA(cudaFuncSetAttribute(k_tc_gemm_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_tc_gemm_tile<<<1, 128, smem, S>>>(tm, a0, b0, (uint32_t)(dpad / KC), idesc16(TM, TN, fp16),
                                      out.p);
  note_launch(ctx, "k_tc_gemm_tile");
  NB_CUDA(cudaMemcpyAsync(out_host, out.p, TM * TN * 4, cudaMemcpyDeviceToHost, S));
  NB_CUDA(cudaStreamSynchronize(S));
}

}  // namespace nb

extern "C" int32_t nomad_b200_debug_tc_gemm(nomad_b200_ctx* ctx, const float* host_rows,
                                            uint64_t rows, uint64_t d, uint32_t a0, uint32_t b0,
                                            float* out128x128) {
  return nb::guard([&] {
    if (!ctx || !host_rows || !out128x128) nb::fail(nb::kParameter, "NULL argument");
    const bool fp16 = (a0 & 0x80000000u) != 0;  // high bit of a0 selects fp16 operands
    a0 &= 0x7FFFFFFFu;
    if (rows < a0 + 128 || rows < b0 + 128) nb::fail(nb::kParameter, "tile out of range");
    nb::bind_device(ctx);
    nb::tc_gemm_tile_check(ctx, host_rows, rows, d, a0, b0, fp16, out128x128);
  });
}
