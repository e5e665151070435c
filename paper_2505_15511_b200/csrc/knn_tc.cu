// kNN fast mode on the 5th-gen tensor cores (knn.hpp:65-109 semantics, bf16
// distances): per cluster, rows are centred on the cluster mean, rounded to
// bf16 into a padded cluster-contiguous copy, and every (query tile,
// candidate tile) product S = A B^T (128 x 128, K = d) runs on tcgen05.mma
// with operands streamed by TMA into 128B-swizzled shared memory (4-stage
// ring) and the fp32 accumulator in TMEM. The epilogue reads the accumulator
// with tcgen05.ld (one thread per query row), forms ||a||^2 + ||b||^2 - 2ab
// and keeps the KP smallest per row. The survivors are re-ranked with the
// reference's exact fp64 distance (knn.cu), so reported distances are exact;
// recall@k against the exact mode measures the bf16 selection.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>

#include "index_common.cuh"
#include "tc_common.cuh"

namespace nb {



namespace {

constexpr int TM = 128;        // query rows per CTA (UMMA M)
constexpr int TN = 128;        // tile width of the diagnostic GEMM
constexpr int KC = 64;         // bf16 columns per stage (one 128B swizzle atom)
constexpr int KPF = 32;        // survivors per query
constexpr uint32_t STAGE_BYTES = (TM + TN) * KC * 2;  // 32 KB

struct TcTile {
  uint32_t row0;   // padded row of this query tile
  uint32_t cbase;  // padded row of the cluster's first member
  uint32_t size;   // cluster size
  uint32_t qoff;   // query offset inside the cluster
};

// bf16(x - mean) into the padded cluster-contiguous copy, fp32 norms.
__global__ void k_tc_prep(const float* __restrict__ x, uint64_t d, uint64_t dpad,
                          const uint32_t* __restrict__ perm_pad, const uint32_t* __restrict__ row_cl,
                          const double* __restrict__ means, uint64_t rows_pad,
                          __nv_bfloat16* __restrict__ xb, float* __restrict__ norms) {
  const uint64_t row = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= rows_pad) return;
  const uint32_t id = perm_pad[row];
  const double* mu = means + (uint64_t)row_cl[row] * d;
  float acc = 0.f;
  for (uint64_t j = lane; j < dpad; j += 32) {
    float v = 0.f;
    if (id != 0xFFFFFFFFu && j < d) v = (float)((double)x[(uint64_t)id * d + j] - mu[j]);
    const __nv_bfloat16 b = __float2bfloat16_rn(v);
    xb[row * dpad + j] = b;
    const float bf = __bfloat162float(b);
    acc = fmaf(bf, bf, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) norms[row] = acc;
}

// v2, warp-specialised: warp 0 = TMA producer, warp 1 = MMA issuer (and TMEM
// owner), warps 2..5 = epilogue (one query row per thread; TMEM lane quarter
// = warp % 4). Candidate tiles are N2 = 256 wide; the fp32 accumulator is
// double-buffered in TMEM (2 x 256 columns) so the epilogue of tile t
// overlaps the MMAs of tile t+1. Each epilogue thread keeps its row's KPF
// best (distance, index) in registers (sorted; insertion is a compare-swap
// chain, rare after the first tiles).
constexpr int TN2 = 256;
constexpr int STAGES2 = 4;
constexpr uint32_t STAGE2_BYTES = (TM + TN2) * KC * 2;  // 48 KB

__global__ void __launch_bounds__(192, 1) k_knn_tc2(const __grid_constant__ CUtensorMap tmap,
                                                    const TcTile* __restrict__ tiles,
                                                    const float* __restrict__ norms,
                                                    const uint32_t* __restrict__ perm_pad,
                                                    uint32_t kchunks, uint32_t* cand_ids,
                                                    float* cand_tau, uint32_t* cand_cnt) {
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
      const uint32_t idesc = tc::idesc_bf16(TM, TN2);
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
    float ld[KPF];
    uint32_t li[KPF];
#pragma unroll
    for (int e = 0; e < KPF; ++e) {
      ld[e] = __int_as_float(0x7f800000);
      li[e] = 0xFFFFFFFFu;
    }
    float tau = ld[KPF - 1];
    for (uint32_t ct = 0; ct < ntiles; ++ct) {
      const uint32_t b = ct & 1;
      float* cnb = cn + b * TN2;
      // candidate norms of this tile (invalid columns -> +inf)
      for (int j = et; j < TN2; j += 128) {
        const uint32_t cl = ct * TN2 + j;
        cnb[j] = cl < T.size ? norms[T.cbase + cl] : __int_as_float(0x7f800000);
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      tc::mbar_wait(&tfull[b], (ct >> 1) & 1);
      tc::fence_after();
      const uint32_t acc = tmem + b * TN2 + ((uint32_t)(q4 * 32) << 16);
#pragma unroll 1
      for (int cc = 0; cc < TN2; cc += 32) {
        float v[32];
        tc::tmem_ld32(acc + cc, v);
        if (!qvalid) continue;
        // distances + below-threshold mask (straight-line); the rare
        // insertions run afterwards from shared memory, one code copy.
        uint32_t mask = 0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float dist = fmaf(-2.f, v[j], qn + cnb[cc + j]);
          if (ct * TN2 + cc + j == q_local) dist = __int_as_float(0x7f800000);
          v[j] = dist;
          mask |= (dist < tau ? 1u : 0u) << j;
        }
        if (mask) {
          float* row = spill + et * 33;
#pragma unroll
          for (int j = 0; j < 32; ++j) row[j] = v[j];
          while (mask) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            float cd = row[j];
            if (!(cd < tau)) continue;
            uint32_t ci = ct * TN2 + cc + j;
#pragma unroll
            for (int e = 0; e < KPF; ++e) {
              if (cd < ld[e]) {
                const float td = ld[e];
                const uint32_t ti = li[e];
                ld[e] = cd;
                li[e] = ci;
                cd = td;
                ci = ti;
              }
            }
            tau = ld[KPF - 1];
          }
        }
      }
      tc::fence_before();
      tc::mbar_arrive(&tempty[b]);
    }
    if (qvalid) {
      const uint32_t gq = perm_pad[T.row0 + r];
      uint32_t c = 0;
#pragma unroll
      for (int e = 0; e < KPF; ++e)
        if (li[e] != 0xFFFFFFFFu) {
          cand_ids[(uint64_t)gq * KPF + c] = perm_pad[T.cbase + li[e]];
          ++c;
        }
      cand_cnt[gq] = c;
      cand_tau[gq] = __int_as_float(0x7f800000);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, 2 * TN2);
}

// Debug / unit path: D = A B^T for one 128 x 128 tile pair (rows a0, b0 of
// the bf16 tensor), written to out[128][128].
__global__ void __launch_bounds__(128, 1) k_tc_gemm_tile(const __grid_constant__ CUtensorMap tmap,
                                                         uint32_t a0, uint32_t b0,
                                                         uint32_t kchunks, float* out) {
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
        tc::umma_bf16(tmem, da + 2 * k, db + 2 * k, tc::idesc_bf16(TM, TN), (kc | k) != 0);
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

CUtensorMap make_tmap(const __nv_bfloat16* xb, uint64_t rows, uint64_t dpad) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof m);
  const cuuint64_t gdim[2] = {dpad, rows};
  const cuuint64_t gstride[1] = {dpad * 2};
  const cuuint32_t box[2] = {KC, TM};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (void*)xb, gdim, gstride,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(kInternal, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return m;
}


}  // namespace

// Fast-mode candidate generation; fills cand_ids[n][32] / cand_cnt[n].
void knn_bf16_candidates(nomad_b200_ctx* ctx, const float* x, uint64_t n, uint64_t d,
                         const uint32_t* assign_d, uint32_t C, DBuf<uint32_t>& cand_ids,
                         DBuf<float>& cand_tau, DBuf<uint32_t>& cand_cnt) {
  cudaStream_t S = ctx->stream;
  DBuf<uint32_t> mem;
  std::vector<uint64_t> off;
  group_by_label(ctx, assign_d, n, C, mem, off);
  // cluster means (centring for bf16)
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
    seq_column_means(ctx, x, d, mem.p, beg, cnt, rows, means.p);
  }
  // padded layout
  std::vector<uint32_t> mem_h(off[C]);
  NB_CUDA(cudaMemcpy(mem_h.data(), mem.p, off[C] * 4, cudaMemcpyDeviceToHost));
  std::vector<uint64_t> pstart(C + 1, 0);
  for (uint32_t r = 0; r < C; ++r) pstart[r + 1] = pstart[r] + (off[r + 1] - off[r] + TM - 1) / TM * TM;
  const uint64_t rows_pad = std::max<uint64_t>(pstart[C], TM);
  if (rows_pad >= (1ull << 31)) fail(kSize, "bf16 kNN: too many rows for TMA coordinates");
  std::vector<uint32_t> perm(rows_pad, 0xFFFFFFFFu), rcl(rows_pad, 0);
  std::vector<TcTile> tiles;
  for (uint32_t r = 0; r < C; ++r) {
    const uint64_t sz = off[r + 1] - off[r];
    for (uint64_t t = 0; t < (pstart[r + 1] - pstart[r]); ++t) rcl[pstart[r] + t] = r;
    for (uint64_t t = 0; t < sz; ++t) perm[pstart[r] + t] = mem_h[off[r] + t];
    if (sz < 2) continue;
    for (uint64_t q = 0; q < sz; q += TM)
      tiles.push_back(TcTile{(uint32_t)(pstart[r] + q), (uint32_t)pstart[r], (uint32_t)sz, (uint32_t)q});
  }
  const uint64_t dpad = (d + KC - 1) / KC * KC;
  DBuf<uint32_t> perm_d(rows_pad), rcl_d(rows_pad);
  NB_CUDA(cudaMemcpyAsync(perm_d.p, perm.data(), rows_pad * 4, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(rcl_d.p, rcl.data(), rows_pad * 4, cudaMemcpyHostToDevice, S));
  DBuf<__nv_bfloat16> xb(rows_pad * dpad);
  DBuf<float> norms(rows_pad);
  k_tc_prep<<<(unsigned)((rows_pad * 32 + 255) / 256), 256, 0, S>>>(x, d, dpad, perm_d.p, rcl_d.p,
                                                                     means.p, rows_pad, xb.p, norms.p);
  note_launch(ctx, "k_tc_prep");
  cand_ids.alloc(n * KPF);
  cand_tau.alloc(n);
  cand_cnt.alloc(n);
  NB_CUDA(cudaMemsetAsync(cand_cnt.p, 0, n * 4, S));
  if (tiles.empty()) return;
  const CUtensorMap tm = make_tmap(xb.p, rows_pad, dpad);
  DBuf<TcTile> tiles_d(tiles.size());
  NB_CUDA(cudaMemcpyAsync(tiles_d.p, tiles.data(), tiles.size() * sizeof(TcTile),
                          cudaMemcpyHostToDevice, S));
  const size_t smem = 1024 + STAGES2 * STAGE2_BYTES + 2 * TN2 * 4 + (2 * STAGES2 + 4) * 8 + 16 +
                      128 * 33 * 4;
  NB_CUDA(cudaFuncSetAttribute(k_knn_tc2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_knn_tc2<<<(unsigned)tiles.size(), 192, smem, S>>>(tm, tiles_d.p, norms.p, perm_d.p,
                                                       (uint32_t)(dpad / KC), cand_ids.p,
                                                       cand_tau.p, cand_cnt.p);
  note_launch(ctx, "k_knn_tc2");
  NB_CUDA(cudaStreamSynchronize(S));
}

// Unit check of the tcgen05 path: rows of a (m x d) f32 host matrix are
// rounded to bf16; returns D = A[a0:a0+128] B[b0:b0+128]^T (fp32, 128 x 128).
void tc_gemm_tile_check(nomad_b200_ctx* ctx, const float* host, uint64_t rows, uint64_t d,
                        uint32_t a0, uint32_t b0, float* out_host) {
  cudaStream_t S = ctx->stream;
  const uint64_t dpad = (d + KC - 1) / KC * KC;
  std::vector<__nv_bfloat16> hb(rows * dpad);
  for (uint64_t i = 0; i < rows; ++i)
    for (uint64_t j = 0; j < dpad; ++j)
      hb[i * dpad + j] = __float2bfloat16_rn(j < d ? host[i * d + j] : 0.f);
  DBuf<__nv_bfloat16> xb(rows * dpad);
  NB_CUDA(cudaMemcpy(xb.p, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice));
  const CUtensorMap tm = make_tmap(xb.p, rows, dpad);
  DBuf<float> out(TM * TN);
  const size_t smem = 1024 + STAGE_BYTES + 64;
  NB_CUDA(cudaFuncSetAttribute(k_tc_gemm_tile, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_tc_gemm_tile<<<1, 128, smem, S>>>(tm, a0, b0, (uint32_t)(dpad / KC), out.p);
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
    if (rows < a0 + 128 || rows < b0 + 128) nb::fail(nb::kParameter, "tile out of range");
    nb::bind_device(ctx);
    nb::tc_gemm_tile_check(ctx, host_rows, rows, d, a0, b0, out128x128);
  });
}
