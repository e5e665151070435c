// Stable grouping by label and exact sequential column means (see
// index_common.cuh).
#include <cub/cub.cuh>

#include "index_common.cuh"

namespace nb {

namespace {

constexpr uint32_t kChunk = 4096;

// Per-chunk label histogram, label-major: hist[label * nchunks + chunk].
__global__ void k_chunk_hist(const uint32_t* labels, uint64_t n, uint32_t L, uint32_t nchunks,
                             uint32_t* hist) {
  extern __shared__ uint32_t h[];
  const bool use_smem = L <= 8192;
  const uint64_t c = blockIdx.x;
  const uint64_t b = c * kChunk, e = umin64(b + kChunk, n);
  if (use_smem) {
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      const uint32_t l = labels[i];
      if (l < L) atomicAdd(&h[l], 1u);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < L; i += blockDim.x) hist[(uint64_t)i * nchunks + c] = h[i];
  } else {
    for (uint64_t i = b + threadIdx.x; i < e; i += blockDim.x) {
      const uint32_t l = labels[i];
      if (l < L) atomicAdd(&hist[(uint64_t)l * nchunks + c], 1u);
    }
  }
}

// One warp per chunk walks its points in order; __match_any_sync ranks equal
// labels inside each 32-point batch, so the scatter preserves id order.
__global__ void k_chunk_scatter(const uint32_t* labels, uint64_t n, uint32_t L, uint32_t nchunks,
                                uint32_t* cursor, uint32_t* members) {
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (warp >= nchunks) return;
  const uint64_t b = (uint64_t)warp * kChunk, e = umin64(b + kChunk, n);
  const uint32_t lt = (1u << lane) - 1u;
  for (uint64_t base = b; base < e; base += 32) {
    const uint64_t i = base + lane;
    const uint32_t l = i < e ? labels[i] : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(0xffffffffu, l);
    const uint32_t rank = __popc(peers & lt);
    const bool leader = (peers >> lane) == 1u;  // highest lane of the group
    uint32_t pos = 0;
    if (l < L) pos = cursor[(uint64_t)l * nchunks + warp] + rank;
    __syncwarp();
    if (l < L && leader) cursor[(uint64_t)l * nchunks + warp] += __popc(peers);
    __syncwarp();
    if (l < L) members[pos] = (uint32_t)i;
  }
}

__global__ void k_extract_offsets(const uint32_t* scanned, const uint32_t* hist, uint32_t L,
                                  uint32_t nchunks, uint64_t* off) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < L) off[r] = scanned[(uint64_t)r * nchunks];
  if (r == L - 1) {
    const uint64_t last = (uint64_t)r * nchunks + nchunks - 1;
    off[L] = (uint64_t)scanned[last] + hist[last];
  }
}

// Same sums, latency-hidden: a CTA per (segment, 32-column group). All 8
// warps stream batches of BR rows (one 128-B row slice per warp instruction,
// cp.async into a double buffer), while warp 0 walks the previous batch in
// order (lanes = columns) with the dependent fp64 adds. Order and rounding
// are exactly k_seq_colsum's (ascending member order, one add per row).
template <int BR>
__global__ void __launch_bounds__(256) k_seq_colsum2(XPtr x, uint64_t d,
                                                     const uint32_t* members,
                                                     const uint64_t* seg_beg,
                                                     const uint64_t* seg_cnt,
                                                     const uint32_t* seg_row, uint32_t nseg,
                                                     double* out, int carry) {
  extern __shared__ float sbuf[];  // [2][BR][33]
  const uint32_t groups = (uint32_t)((d + 31) / 32);
  const uint32_t sidx = blockIdx.x / groups;
  const uint64_t j0 = (uint64_t)(blockIdx.x % groups) * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t beg = seg_beg[sidx], cnt = seg_cnt[sidx];
  if (cnt == 0) return;
  const uint64_t j = j0 + lane;
  const bool colok = j < d;
  auto issue = [&](uint64_t b) {
    const uint64_t r0 = b * BR;
    float* dst = sbuf + (b & 1) * BR * 33;
    for (int rr = warp; rr < BR; rr += 8) {
      const uint64_t t = r0 + rr;
      if (t < cnt && colok) {
        const uint64_t row = members ? members[beg + t] : beg + t;
        if (x.bf) {  // 2-byte elements: plain load, widened into the buffer
          dst[rr * 33 + lane] = x[row * d + j];
        } else {
          const uint32_t sa = (uint32_t)__cvta_generic_to_shared(dst + rr * 33 + lane);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa),
                       "l"(static_cast<const float*>(x.p) + row * d + j)
                       : "memory");
        }
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const uint64_t nb = (cnt + BR - 1) / BR;
  // carry: continue the running sums already in `out` (the previous rank's,
  // row-sharded build) and leave them undivided
  double acc = (carry && colok) ? out[(uint64_t)seg_row[sidx] * d + j] : 0.0;
  issue(0);
  for (uint64_t b = 0; b < nb; ++b) {
    if (b + 1 < nb) issue(b + 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      const float* src = sbuf + (b & 1) * BR * 33;
      const int m = (int)umin64(BR, cnt - b * BR);
      for (int r = 0; r < m; ++r) acc = __dadd_rn(acc, colok ? (double)src[r * 33 + lane] : 0.0);
    }
    __syncthreads();
  }
  if (warp == 0 && colok)
    out[(uint64_t)seg_row[sidx] * d + j] = carry ? acc : __ddiv_rn(acc, (double)cnt);
}

}  // namespace

void group_by_label(nomad_b200_ctx* ctx, const uint32_t* labels, uint64_t n, uint32_t L,
                    DBuf<uint32_t>& members, std::vector<uint64_t>& off) {
  cudaStream_t S = ctx->stream;
  const uint32_t nchunks = (uint32_t)((n + kChunk - 1) / kChunk);
  const uint64_t H = (uint64_t)L * nchunks;
  DBuf<uint32_t> hist(H), scanned(H);
  NB_CUDA(cudaMemsetAsync(hist.p, 0, H * 4, S));
  k_chunk_hist<<<nchunks, 256, L <= 8192 ? L * 4 : 0, S>>>(labels, n, L, nchunks, hist.p);
  note_launch(ctx, "k_chunk_hist");
  size_t tmp = 0;
  NB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, hist.p, scanned.p, (int64_t)H, S));
  DBuf<uint8_t> tb(tmp + 1);
  NB_CUDA(cub::DeviceScan::ExclusiveSum(tb.p, tmp, hist.p, scanned.p, (int64_t)H, S));
  note_launch(ctx, "cub_exclusive_sum");
  DBuf<uint64_t> offd(L + 1);
  k_extract_offsets<<<(L + 255) / 256, 256, 0, S>>>(scanned.p, hist.p, L, nchunks, offd.p);
  note_launch(ctx, "k_extract_offsets");
  off.assign(L + 1, 0);
  NB_CUDA(cudaMemcpyAsync(off.data(), offd.p, (L + 1) * 8, cudaMemcpyDeviceToHost, S));
  NB_CUDA(cudaStreamSynchronize(S));
  members.alloc(std::max<uint64_t>(off[L], 1));
  // scanned now serves as the per-(label, chunk) write cursor
  k_chunk_scatter<<<(nchunks * 32 + 255) / 256, 256, 0, S>>>(labels, n, L, nchunks, scanned.p,
                                                              members.p);
  note_launch(ctx, "k_chunk_scatter");
}

void seq_column_means(nomad_b200_ctx* ctx, XPtr x, uint64_t d, const uint32_t* members,
                      const std::vector<uint64_t>& beg, const std::vector<uint64_t>& cnt,
                      const std::vector<uint32_t>& seg_ids, double* out, bool carry) {
  cudaStream_t S = ctx->stream;
  const uint32_t nseg = (uint32_t)seg_ids.size();
  if (!nseg) return;
  DBuf<uint64_t> db(nseg), dc(nseg);
  DBuf<uint32_t> dr(nseg);
  NB_CUDA(cudaMemcpyAsync(db.p, beg.data(), nseg * 8, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(dc.p, cnt.data(), nseg * 8, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(dr.p, seg_ids.data(), nseg * 4, cudaMemcpyHostToDevice, S));
  const uint64_t ctas = (uint64_t)nseg * ((d + 31) / 32);
  constexpr int BR = 256;
  const size_t smem = 2 * BR * 33 * sizeof(float);
  NB_CUDA(cudaFuncSetAttribute(k_seq_colsum2<BR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  k_seq_colsum2<BR><<<(unsigned)ctas, 256, smem, S>>>(x, d, members, db.p, dc.p, dr.p, nseg, out,
                                                      carry ? 1 : 0);
  note_launch(ctx, "k_seq_colsum2");
  NB_CUDA(cudaStreamSynchronize(S));
}

// ---- fast_column_means: deterministic parallel form (fixed 1024-row chunks,
// chunk sums added in chunk order) for centres whose exact value does not
// matter, only that it is fixed: the tensor-core kNN centring and the
// sub-cluster certificate centres (knn_tc.cu, knn.cu). One CTA per chunk, one
// column per thread, rows walked in order.
namespace {
constexpr uint32_t kMeanChunk = 1024;

__global__ void k_chunk_colsum(XPtr x, uint32_t d, const uint32_t* __restrict__ members,
                               const uint64_t* __restrict__ cbeg, const uint32_t* __restrict__ ccnt,
                               double* __restrict__ part) {
  const uint64_t b = cbeg[blockIdx.x];
  const uint32_t c = ccnt[blockIdx.x];
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    uint32_t i = 0;
    for (; i + 4 <= c; i += 4) {
      const uint64_t r0 = members ? members[b + i] : b + i;
      const uint64_t r1 = members ? members[b + i + 1] : b + i + 1;
      const uint64_t r2 = members ? members[b + i + 2] : b + i + 2;
      const uint64_t r3 = members ? members[b + i + 3] : b + i + 3;
      a0 += (double)x[r0 * d + j];
      a1 += (double)x[r1 * d + j];
      a2 += (double)x[r2 * d + j];
      a3 += (double)x[r3 * d + j];
    }
    for (; i < c; ++i) a0 += (double)x[(members ? members[b + i] : b + i) * (uint64_t)d + j];
    part[(uint64_t)blockIdx.x * d + j] = (a0 + a1) + (a2 + a3);
  }
}

__global__ void k_chunk_means(uint32_t d, const double* __restrict__ part,
                              const uint32_t* __restrict__ sfirst, const uint32_t* __restrict__ snum,
                              const uint64_t* __restrict__ scnt, const uint32_t* __restrict__ sid,
                              double* __restrict__ out) {
  const uint32_t s = blockIdx.x;
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) {
    double a = 0.0;
    for (uint32_t t = 0; t < snum[s]; ++t) a += part[(uint64_t)(sfirst[s] + t) * d + j];
    out[(uint64_t)sid[s] * d + j] = a / (double)scnt[s];
  }
}
}  // namespace

void fast_column_means(nomad_b200_ctx* ctx, XPtr x, uint64_t d, const uint32_t* members,
                       const std::vector<uint64_t>& beg, const std::vector<uint64_t>& cnt,
                       const std::vector<uint32_t>& seg_ids, double* out) {
  cudaStream_t S = ctx->stream;
  std::vector<uint64_t> cb;
  std::vector<uint32_t> cc, sfirst, snum, sid;
  std::vector<uint64_t> scnt;
  for (size_t s = 0; s < seg_ids.size(); ++s) {
    if (!cnt[s]) continue;
    sfirst.push_back((uint32_t)cb.size());
    for (uint64_t o = 0; o < cnt[s]; o += kMeanChunk) {
      cb.push_back(beg[s] + o);
      cc.push_back((uint32_t)std::min<uint64_t>(kMeanChunk, cnt[s] - o));
    }
    snum.push_back((uint32_t)(cb.size() - sfirst.back()));
    scnt.push_back(cnt[s]);
    sid.push_back(seg_ids[s]);
  }
  if (cb.empty()) return;
  const uint32_t nch = (uint32_t)cb.size(), nseg = (uint32_t)sid.size();
  DBuf<uint64_t> cb_d(nch), scnt_d(nseg);
  DBuf<uint32_t> cc_d(nch), sf_d(nseg), sn_d(nseg), sid_d(nseg);
  DBuf<double> part((uint64_t)nch * d);
  NB_CUDA(cudaMemcpyAsync(cb_d.p, cb.data(), nch * 8, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(cc_d.p, cc.data(), nch * 4, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(sf_d.p, sfirst.data(), nseg * 4, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(sn_d.p, snum.data(), nseg * 4, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(scnt_d.p, scnt.data(), nseg * 8, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(sid_d.p, sid.data(), nseg * 4, cudaMemcpyHostToDevice, S));
  const unsigned th = (unsigned)std::min<uint64_t>(256, (d + 31) / 32 * 32);
  k_chunk_colsum<<<nch, th, 0, S>>>(x, (uint32_t)d, members, cb_d.p, cc_d.p, part.p);
  note_launch(ctx, "k_chunk_colsum");
  k_chunk_means<<<nseg, th, 0, S>>>((uint32_t)d, part.p, sf_d.p, sn_d.p, scnt_d.p, sid_d.p, out);
  note_launch(ctx, "k_chunk_means");
  NB_CUDA(cudaStreamSynchronize(S));
}

}  // namespace nb
