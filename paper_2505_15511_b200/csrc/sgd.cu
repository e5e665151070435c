// SGD epoch kernels and cluster-means kernels (see sgd_kernels.cuh).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "sgd_device.cuh"
#include "sgd_kernels.cuh"

namespace nb {

// Sequential fp64 sum of p[0], p[stride], ..., p[(m-1) stride] in that order
// by one warp (the reference's accumulation order; lane 0 holds the result).
// The warp stages 256 values in shared memory, and while lane 0 adds them
// (loads ahead of the dependent adds: the chain runs at DADD latency, ~8
// cycles) the next 256 are already in flight into every lane's registers.
__device__ __forceinline__ double warp_seq_sum(const double* __restrict__ p, size_t stride,
                                               uint32_t m, double* buf) {
  const uint32_t lane = threadIdx.x & 31;
  double acc = 0.0;
  double nx[8];
  auto fetch = [&](uint32_t b0) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t e = b0 + lane + 32 * u;
      nx[u] = e < m ? p[stride * e] : 0.0;
    }
  };
  fetch(0);
  for (uint32_t b0 = 0; b0 < m; b0 += 256) {
#pragma unroll
    for (int u = 0; u < 8; ++u) buf[lane + 32 * u] = nx[u];
    __syncwarp();
    if (b0 + 256 < m) fetch(b0 + 256);  // in flight during the adds below
    if (lane == 0) {
      const uint32_t n = min(256u, m - b0);
      uint32_t e = 0;
      for (; e + 8 <= n; e += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = buf[e + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, v[u]);
      }
      for (; e < n; ++e) acc = __dadd_rn(acc, buf[e]);
    }
    __syncwarp();
  }
  return acc;
}

// Per-worker loss in sequential draw order (optimizer.hpp:289-290), one warp
// per worker.
__global__ void k_loss_seq(const double* slot, const uint32_t* base, const WorkerDev* wk,
                           uint32_t nw, double* out) {
  __shared__ double buf[4][256];
  const uint32_t wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t w = blockIdx.x * (blockDim.x >> 5) + wi;
  if (w >= nw) return;
  const double acc = warp_seq_sum(slot + base[w], 1, wk[w].draws, buf[wi]);
  if (lane == 0) out[w] = acc;
}

// ------------------------------------------------------ K9 cluster means
//
// Exact: per local cluster and coordinate, a sequential sum over the
// cluster's contiguous segment (ascending original id == the order of
// gather_means, optimizer.hpp:163-168 / :420-428), then / count; one warp
// per (cluster, coordinate) chain.
__global__ void k_means_exact(const double2* pos, const LocalCluster* lc, uint32_t ncl,
                              double* slot /* ncl x 2 */) {
  __shared__ double buf[4][256];
  const uint32_t wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t g = blockIdx.x * (blockDim.x >> 5) + wi;
  if (g >= 2 * ncl) return;
  const uint32_t c = g >> 1, dim = g & 1;
  const LocalCluster L = lc[c];
  const double* p = reinterpret_cast<const double*>(pos) + 2 * (size_t)L.start + dim;
  const double acc = warp_seq_sum(p, 2, L.count, buf[wi]);
  if (lane == 0) slot[g] = __ddiv_rn(acc, (double)L.count);
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

void launch_loss_seq(const double* slot, const uint32_t* base, const WorkerDev* wk, uint32_t nw,
                     double* out, cudaStream_t st) {
  k_loss_seq<<<blocks_for(nw, 4), 128, 0, st>>>(slot, base, wk, nw, out);
}

void launch_means_exact(const double2* pos, const LocalCluster* lc, uint32_t ncl, double* slot,
                        cudaStream_t st) {
  k_means_exact<<<blocks_for(2 * ncl, 4), 128, 0, st>>>(pos, lc, ncl, slot);
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
