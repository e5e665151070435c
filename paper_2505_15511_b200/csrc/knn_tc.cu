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
constexpr int TN = 128;        // candidate rows per tile (UMMA N)
constexpr int KC = 64;         // bf16 columns per stage (one 128B swizzle atom)
constexpr int STAGES = 4;
constexpr int KPF = 32;        // survivors per query
constexpr int CAPF = 64;       // per-row buffer
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

__device__ void row_compact(float* bd, uint32_t* bi, int r, uint32_t& cnt, float& tau) {
  // keep the KPF smallest of cnt entries (column-major row r), selection sort
  for (int i = 0; i < KPF; ++i) {
    int m = i;
    float mv = bd[i * TM + r];
    for (uint32_t e = i + 1; e < cnt; ++e) {
      const float v = bd[e * TM + r];
      if (v < mv) { mv = v; m = (int)e; }
    }
    if (m != i) {
      const float tv = bd[i * TM + r];
      const uint32_t ti = bi[i * TM + r];
      bd[i * TM + r] = mv;
      bi[i * TM + r] = bi[m * TM + r];
      bd[m * TM + r] = tv;
      bi[m * TM + r] = ti;
    }
  }
  cnt = KPF;
  tau = bd[(KPF - 1) * TM + r];
}

__global__ void __launch_bounds__(128, 1) k_knn_tc(const __grid_constant__ CUtensorMap tmap,
                                                   const TcTile* __restrict__ tiles,
                                                   const float* __restrict__ norms,
                                                   const uint32_t* __restrict__ perm_pad,
                                                   uint32_t kchunks, uint32_t* cand_ids,
                                                   float* cand_tau, uint32_t* cand_cnt) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* base = smem + ((1024 - (tc::smem_u32(smem) & 1023)) & 1023);
  uint8_t* stage_mem = base;                                  // STAGES x 32 KB
  float* bd = reinterpret_cast<float*>(base + STAGES * STAGE_BYTES);  // CAPF x TM
  uint32_t* bi = reinterpret_cast<uint32_t*>(bd + CAPF * TM);
  uint64_t* full = reinterpret_cast<uint64_t*>(bi + CAPF * TM);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const TcTile T = tiles[blockIdx.x];
  const int r = threadIdx.x, warp = r >> 5;
  if (warp == 0) tc::tmem_alloc(tmem_slot, TN);
  if (r == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(done, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  const uint32_t q_local = T.qoff + r;  // my query inside the cluster
  const bool qvalid = q_local < T.size;
  const float qn = norms[T.row0 + r];
  uint32_t cnt = 0;
  float tau = __int_as_float(0x7f800000);
  const uint32_t ntiles = (T.size + TN - 1) / TN;
  const uint32_t total = ntiles * kchunks;
  const uint32_t idesc = tc::idesc_bf16(TM, TN);
  uint32_t issued = 0;  // TMA loads issued (thread 0)
  for (uint32_t ct = 0; ct < ntiles; ++ct) {
    if (r == 0) {
      for (uint32_t kc = 0; kc < kchunks; ++kc) {
        const uint32_t it = ct * kchunks + kc;
        // keep the TMA producer up to STAGES loads ahead of the MMA
        while (issued < total && issued < it + STAGES) {
          const uint32_t s = issued % STAGES;
          if (issued >= STAGES) tc::mbar_wait(&empty[s], ((issued / STAGES) - 1) & 1);
          const uint32_t ict = issued / kchunks, ikc = issued % kchunks;
          uint8_t* sa = stage_mem + s * STAGE_BYTES;
          tc::mbar_expect_tx(&full[s], STAGE_BYTES);
          tc::tma_load_2d(sa, &tmap, &full[s], (int32_t)(ikc * KC), (int32_t)T.row0);
          tc::tma_load_2d(sa + TM * KC * 2, &tmap, &full[s], (int32_t)(ikc * KC),
                          (int32_t)(T.cbase + ict * TN));
          ++issued;
        }
        const uint32_t s = it % STAGES;
        tc::mbar_wait(&full[s], (it / STAGES) & 1);
        tc::fence_after();
        const uint32_t sa = tc::smem_u32(stage_mem + s * STAGE_BYTES);
        const uint64_t da = tc::sdesc_k_sw128(sa), db = tc::sdesc_k_sw128(sa + TM * KC * 2);
#pragma unroll
        for (int k = 0; k < KC / 16; ++k)
          tc::umma_bf16(tmem, da + 2 * k, db + 2 * k, idesc, (kc | k) != 0);
        tc::umma_commit(&empty[s]);
      }
      tc::umma_commit(done);
    }
    __syncwarp();
    tc::mbar_wait(done, ct & 1);
    tc::fence_after();
    // epilogue: my TMEM lane = my query row; 4 x 32 columns
#pragma unroll 1
    for (int cc = 0; cc < TN; cc += 32) {
      float v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + cc, v);
      if (!qvalid) continue;
      const uint32_t c0 = ct * TN + cc;  // cluster-local index of column 0
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const uint32_t cl = c0 + j;
        if (cl >= T.size || cl == q_local) continue;
        const float dist = qn + norms[T.cbase + cl] - 2.f * v[j];
        if (dist < tau) {
          bd[cnt * TM + r] = dist;
          bi[cnt * TM + r] = cl;
          if (++cnt == CAPF) row_compact(bd, bi, r, cnt, tau);
        }
      }
    }
    tc::fence_before();
    __syncthreads();
  }
  if (qvalid) {
    if (cnt > KPF) row_compact(bd, bi, r, cnt, tau);
    const uint32_t gq = perm_pad[T.row0 + r];
    for (uint32_t e = 0; e < cnt; ++e) cand_ids[(uint64_t)gq * KPF + e] = perm_pad[T.cbase + bi[e * TM + r]];
    cand_cnt[gq] = cnt;
    cand_tau[gq] = __int_as_float(0x7f800000);
  }
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, TN);
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

size_t knn_tc_smem() {
  return 1024 + STAGES * STAGE_BYTES + (size_t)CAPF * TM * 8 + (2 * STAGES + 1) * 8 + 16;
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
  const size_t smem = knn_tc_smem();
  NB_CUDA(cudaFuncSetAttribute(k_knn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k_knn_tc<<<(unsigned)tiles.size(), 128, smem, S>>>(tm, tiles_d.p, norms.p, perm_d.p,
                                                      (uint32_t)(dpad / KC), cand_ids.p, cand_tau.p,
                                                      cand_cnt.p);
  note_launch(ctx, "k_knn_tc");
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
