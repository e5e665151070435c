// PCA initialisation (pca.hpp:79-218) on the GPU, bit-exact: both data
// passes of covariance_apply (pca.hpp:34-55) follow the reference's
// summation order — t_i is a j-ascending chain per row (thread per row, rows
// staged through shared memory), y_j an i-ascending chain per column
// (cp.async-staged column chains) — with _rn intrinsics (no FMA); the
// d-dimensional vector algebra (deflation, normalisation, drift test, 2x2
// Rayleigh-Ritz, sign rule) runs on the host in the reference's expression
// order; the projection, column means and variances are again sequential
// chains. The start vectors and the rank-1 jitter come from the reference's
// own "pca" Rng stream.
#include <algorithm>
#include <cmath>
#include <exception>
#include <memory>
#include <thread>

#include "index_common.cuh"
#include "shard.cuh"

namespace nb {

namespace {

// t_i = sum_{j ascending} ((double)x_ij - mean_j) * v_j   (pca.hpp:40-45)
// thread per row; a 128-row x 32-column tile is staged through shared memory.
__global__ void __launch_bounds__(128) k_pca_rows(XPtr x, uint64_t n,
                                                  uint32_t d, const double* __restrict__ mean,
                                                  const double* __restrict__ v,
                                                  double* __restrict__ t, double* __restrict__ t2,
                                                  const double* __restrict__ v2) {
  constexpr int TP = 128, DK = 32;
  __shared__ float xs[TP][DK + 1];
  __shared__ double ms[DK], vs[DK], vs2[DK];
  const uint64_t p0 = (uint64_t)blockIdx.x * TP;
  const uint64_t gp = p0 + threadIdx.x;
  double acc = 0.0, acc2 = 0.0;
  for (uint32_t j0 = 0; j0 < d; j0 += DK) {
    __syncthreads();
    for (int e = threadIdx.x; e < TP * DK; e += TP) {
      const int p = e / DK, jj = e % DK;
      const uint64_t q = p0 + p;
      xs[p][jj] = (q < n && j0 + jj < d) ? x[q * d + j0 + jj] : 0.f;
    }
    if (threadIdx.x < DK && j0 + threadIdx.x < d) {
      ms[threadIdx.x] = mean[j0 + threadIdx.x];
      vs[threadIdx.x] = v[j0 + threadIdx.x];
      if (v2) vs2[threadIdx.x] = v2[j0 + threadIdx.x];
    }
    __syncthreads();
    const int jmax = min(DK, (int)(d - j0));
    for (int jj = 0; jj < jmax; ++jj) {
      const double c = __dsub_rn((double)xs[threadIdx.x][jj], ms[jj]);
      acc = __dadd_rn(acc, __dmul_rn(c, vs[jj]));
      if (v2) acc2 = __dadd_rn(acc2, __dmul_rn(c, vs2[jj]));
    }
  }
  if (gp < n) {
    t[gp * (t2 ? 2 : 1)] = acc;
    if (t2) t2[gp * 2] = acc2;
  }
}

// y_j = (sum_{i ascending} ((double)x_ij - mean_j) * t_i) / n   (pca.hpp:47-54)
// CTA per 32-column group: 8 warps stream BR-row slices (cp.async, double
// buffer) and t; warp 0 runs the 32 column chains in order.
// carry: y holds running sums (a row-sharded carry chain): continue them and
// store them undivided.
template <int BR>
__global__ void __launch_bounds__(256) k_pca_cols(XPtr x, uint64_t n,
                                                  uint32_t d, const double* __restrict__ mean,
                                                  const double* __restrict__ t,
                                                  double* __restrict__ y, int carry) {
  extern __shared__ float sbuf[];  // [2][BR][33]
  __shared__ double ts[2][BR];
  const uint64_t j0 = (uint64_t)blockIdx.x * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t j = j0 + lane;
  const bool colok = j < d;
  auto issue = [&](uint64_t b) {
    const uint64_t r0 = b * BR;
    float* dst = sbuf + (b & 1) * BR * 33;
    for (int rr = warp; rr < BR; rr += 8) {
      const uint64_t row = r0 + rr;
      if (row < n && colok) {
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
    for (int rr = threadIdx.x; rr < BR; rr += 256)
      if (r0 + rr < n) ts[b & 1][rr] = t[r0 + rr];
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const uint64_t nb = (n + BR - 1) / BR;
  const double m = colok ? mean[j] : 0.0;
  double acc = (carry && colok) ? y[j] : 0.0;
  issue(0);
  for (uint64_t b = 0; b < nb; ++b) {
    if (b + 1 < nb) issue(b + 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    if (warp == 0 && colok) {
      const float* src = sbuf + (b & 1) * BR * 33;
      const double* tb = ts[b & 1];
      const int mrows = (int)umin64(BR, n - b * BR);
      int r = 0;
      for (; r + 8 <= mrows; r += 8) {  // products ahead of the in-order adds
        double p[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          p[u] = __dmul_rn(__dsub_rn((double)src[(r + u) * 33 + lane], m), tb[r + u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __dadd_rn(acc, p[u]);
      }
      for (; r < mrows; ++r)
        acc = __dadd_rn(acc, __dmul_rn(__dsub_rn((double)src[r * 33 + lane], m), tb[r]));
    }
    __syncthreads();
  }
  if (warp == 0 && colok) y[j] = carry ? acc : __ddiv_rn(acc, (double)n);
}

__global__ void k_div_vec(double* v, uint32_t d, double n) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < d) v[j] = __ddiv_rn(v[j], n);
}

// Sequential chains over a strided column of the layout (pca.hpp:197-212):
// mode 0: sum_i v_i; mode 1: sum_i (v_i - mu)^2. One adding thread; the
// block stages the next tile.
__global__ void k_seq_col(const double* lay, uint64_t n, int comp, int mode, double mu,
                          double* out, int carry) {
  constexpr int T = 2048;
  __shared__ double buf[2][T];
  double acc = carry ? *out : 0.0;  // carry: continue the previous rank's chain
  int cur = 0;
  for (uint64_t e = threadIdx.x; e < T && e < n; e += blockDim.x) buf[0][e] = lay[2 * e + comp];
  __syncthreads();
  for (uint64_t b = 0; b < n; b += T) {
    const uint64_t nb = b + T;
    for (uint64_t e = threadIdx.x; e < T && nb + e < n; e += blockDim.x)
      buf[cur ^ 1][e] = lay[2 * (nb + e) + comp];
    if (threadIdx.x == 0) {
      const uint64_t m = umin64(T, n - b);
      if (mode == 0) {
        for (uint64_t e = 0; e < m; ++e) acc = __dadd_rn(acc, buf[cur][e]);
      } else {
        for (uint64_t e = 0; e < m; ++e) {
          const double c = __dsub_rn(buf[cur][e], mu);
          acc = __dadd_rn(acc, __dmul_rn(c, c));
        }
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  if (threadIdx.x == 0) *out = acc;
}

// sums of (x - mean)^2 and x^2 over all entries; column sums / sq of layout
__global__ void k_pca_moments(XPtr x, uint64_t N, uint32_t d,
                              const double* __restrict__ mean, double* out2) {
  double v = 0.0, s = 0.0;
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < N;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const double xv = (double)x[e];
    const double c = xv - mean[e % d];
    v += c * c;
    s += xv * xv;
  }
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out2[0], v);
    atomicAdd(&out2[1], s);
  }
}

__global__ void k_layout_scale(double* lay, uint64_t n, int comp, double sd) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    lay[2 * i + comp] /= sd;
}

__global__ void k_layout_set(double* lay, uint64_t n, int comp, const double* v) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    lay[2 * i + comp] = v[i];
}

// Covariance sums S = X_c^T X_c (fast PCA): grid (upper-triangle 32x32 tiles,
// row slices); each CTA accumulates its tile over its row slice in fp64
// (thread = 4 entries of one column), 64 centred rows staged per step;
// partials are summed per entry in slice order by k_cov_reduce
// (deterministic).
constexpr int CV_ROWS = 64;
__global__ void __launch_bounds__(256) k_cov_partial(XPtr x, uint64_t n,
                                                     uint32_t d, const double* __restrict__ mean,
                                                     const uint2* __restrict__ tiles,
                                                     uint32_t slices, double* __restrict__ part) {
  __shared__ double A[CV_ROWS][33], B[CV_ROWS][33];
  const uint2 T = tiles[blockIdx.x];  // (row tile, col tile), row <= col
  const uint32_t i0 = T.x * 32, j0 = T.y * 32;
  const uint32_t sl = blockIdx.y;
  const uint64_t r0 = n * sl / slices, r1 = n * (sl + 1) / slices;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (uint64_t rb = r0; rb < r1; rb += CV_ROWS) {
    __syncthreads();
    for (int e = threadIdx.x; e < CV_ROWS * 32; e += 256) {
      const int rr = e >> 5, cc = e & 31;
      const uint64_t row = rb + rr;
      const bool ok = row < r1;
      A[rr][cc] = (ok && i0 + cc < d) ? (double)x[row * d + i0 + cc] - mean[i0 + cc] : 0.0;
      B[rr][cc] = (ok && j0 + cc < d) ? (double)x[row * d + j0 + cc] - mean[j0 + cc] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < CV_ROWS; ++rr) {
      const double bv = B[rr][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = fma(A[rr][ty + 8 * q], bv, acc[q]);
    }
  }
  const uint64_t base = ((uint64_t)blockIdx.x * slices + sl) * 1024;
#pragma unroll
  for (int q = 0; q < 4; ++q) part[base + (ty + 8 * q) * 32 + tx] = acc[q];
}

// C[i][j] (full symmetric, row-major) = sum over slices of the tile partials.
__global__ void k_cov_reduce(const double* __restrict__ part, const uint2* __restrict__ tiles,
                             uint32_t ntiles, uint32_t slices, uint32_t d, double* __restrict__ C) {
  const uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (g >= (uint64_t)ntiles * 1024) return;
  const uint32_t t = (uint32_t)(g >> 10), e = (uint32_t)(g & 1023);
  const uint32_t i = tiles[t].x * 32 + (e >> 5), j = tiles[t].y * 32 + (e & 31);
  if (i >= d || j >= d) return;
  double s = 0.0;
  for (uint32_t sl = 0; sl < slices; ++sl) s += part[((uint64_t)t * slices + sl) * 1024 + e];
  C[(uint64_t)i * d + j] = s;
  C[(uint64_t)j * d + i] = s;
}

// y = C v / n, one warp per output entry (fixed-order lane sums + butterfly).
__global__ void k_cov_apply(const double* __restrict__ C, const double* __restrict__ v, uint32_t d,
                            double inv_n, double* __restrict__ y) {
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= d) return;
  double s = 0.0;
  for (uint32_t j = lane; j < d; j += 32) s = fma(C[(uint64_t)i * d + j], v[j], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[i] = s * inv_n;
}

double dot(const std::vector<double>& a, const std::vector<double>& b) {
  double acc = 0.0;
  for (size_t j = 0; j < a.size(); ++j) acc += a[j] * b[j];
  return acc;
}
double normalize(std::vector<double>& v) {
  const double norm = std::sqrt(dot(v, v));
  if (norm > 0.0)
    for (double& x : v) x /= norm;
  return norm;
}

}  // namespace

// S = X_c^T X_c (d x d, fp64, row-major, symmetric) of the centred data.
void covariance_sums(nomad_b200_ctx* ctx, XPtr x, uint64_t n, uint64_t d,
                     const double* mean, double* cov) {
  cudaStream_t S = ctx->stream;
  const uint32_t nt = (uint32_t)((d + 31) / 32);
  std::vector<uint2> th;
  for (uint32_t a = 0; a < nt; ++a)
    for (uint32_t b = a; b < nt; ++b) th.push_back(make_uint2(a, b));
  const uint32_t ntl = (uint32_t)th.size();
  // enough CTAs to cover the GPU; each slice keeps >= 1024 rows
  uint32_t slices = std::max<uint32_t>(1, (uint32_t)((4ull * ctx->sm_count + ntl - 1) / ntl));
  slices = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(slices, n / 1024));
  DBuf<uint2> tiles_d(ntl);
  NB_CUDA(cudaMemcpyAsync(tiles_d.p, th.data(), ntl * sizeof(uint2), cudaMemcpyHostToDevice, S));
  DBuf<double> part((uint64_t)ntl * slices * 1024);
  k_cov_partial<<<dim3(ntl, slices), 256, 0, S>>>(x, n, (uint32_t)d, mean, tiles_d.p, slices,
                                                 part.p);
  note_launch(ctx, "k_cov_partial");
  k_cov_reduce<<<(unsigned)(((uint64_t)ntl * 1024 + 255) / 256), 256, 0, S>>>(
      part.p, tiles_d.p, ntl, slices, (uint32_t)d, cov);
  note_launch(ctx, "k_cov_reduce");
  NB_CUDA(cudaStreamSynchronize(S));
}

// layout_out: device n x 2.
// fast == false: every covariance apply is the reference's two-pass
// X_c^T (X_c v) / n with its summation orders (bit-identical result).
// fast == true: the covariance sums S = X_c^T X_c are formed once (fp64,
// k_cov_partial / k_cov_reduce) and each apply is S v / n; the power
// iteration, deflation, Rayleigh-Ritz step, sign rule and standardisation are
// unchanged. The basis agrees with the reference's to rounding, so the layout
// spans the reference's principal plane; its in-plane orientation can differ:
// pca.hpp:150-165 rotates the converged basis by atan2(eigen0 - h00, h01),
// two quantities that are both at rounding-noise level once the power
// iteration has converged, so only the bit-exact path reproduces the
// reference's orientation.
//
// Row-sharded (comm != nullptr): this rank holds rows
// [row0, row0 + n) of an N-row dataset and writes their layout rows. Every
// ascending-row sum — the data mean, each exact covariance apply's column
// chains, the layout's column mean and spread — is a carry chain over the
// ranks (shard.cuh), so the exact form is bit-identical to one GPU; the fast
// form's covariance sums are added over the ranks in rank order; the
// zero-variance test's moments likewise; the host-side vector algebra runs
// identically on every rank; rank r skips the first row0 jitter draws.
void pca_init_dev(nomad_b200_ctx* ctx, XPtr x, uint64_t n, uint64_t d, uint64_t seed,
                  double* layout_out, bool fast, Comm* comm = nullptr, uint64_t row0 = 0,
                  uint64_t N = 0) {
  cudaStream_t S = ctx->stream;
  if (!comm) N = n;
  if (N < 2) fail(kParameter, "need at least 2 rows");
  HostRng rng(HostRng::stream_seed(seed, 0x706361 /* "pca" */));
  DBuf<double> mean(d), vd(d), yd(d), t(std::max<uint64_t>(n, 1)), mom(2);
  if (!comm) {
    seq_column_means(ctx, x, d, nullptr, {0}, {n}, {0}, mean.p);  // pca.hpp:84-89
  } else {
    comm->chain(mean.p, d, [&] {
      if (n) seq_column_means(ctx, x, d, nullptr, {0}, {n}, {0}, mean.p, true);
    });
    k_div_vec<<<(unsigned)((d + 255) / 256), 256, 0, S>>>(mean.p, (uint32_t)d, (double)N);
    note_launch(ctx, "k_div_vec");
  }
  NB_CUDA(cudaMemsetAsync(mom.p, 0, 16, S));
  if (n) {
    k_pca_moments<<<ctx->sm_count * 8, 256, 0, S>>>(x, n * d, (uint32_t)d, mean.p, mom.p);
    note_launch(ctx, "k_pca_moments");
  }
  double mh[2];
  NB_CUDA(cudaMemcpyAsync(mh, mom.p, 16, cudaMemcpyDeviceToHost, S));
  NB_CUDA(cudaStreamSynchronize(S));
  if (comm) {  // rank-order sums of the ranks' moments
    std::vector<double> all(2 * (size_t)comm->world);
    comm->allgather(mh, 16, all.data());
    mh[0] = mh[1] = 0.0;
    for (int r = 0; r < comm->world; ++r) {
      mh[0] += all[2 * r];
      mh[1] += all[2 * r + 1];
    }
  }
  const double total_var = mh[0] / static_cast<double>(N);
  const double total_sq = mh[1] / static_cast<double>(N);
  if (total_var <= 1e-18 * std::max(1.0, total_sq))
    fail(kDegenerate, "data has zero variance");

  const unsigned row_blocks = (unsigned)((n + 127) / 128);
  constexpr int BR = 256;
  const size_t col_smem = 2 * BR * 33 * sizeof(float);
  NB_CUDA(cudaFuncSetAttribute(k_pca_cols<BR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)col_smem));
  DBuf<double> cov;
  if (fast) {
    cov.alloc(d * d);
    if (n) covariance_sums(ctx, x, n, d, mean.p, cov.p);
    else NB_CUDA(cudaMemsetAsync(cov.p, 0, d * d * 8, S));
    if (comm) {  // S = sum over ranks in rank order
      std::vector<double> mine(d * d), all((size_t)comm->world * d * d);
      NB_CUDA(cudaMemcpyAsync(mine.data(), cov.p, d * d * 8, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
      comm->allgather(mine.data(), d * d * 8, all.data());
      for (size_t e = 0; e < d * d; ++e) {
        double acc = all[e];
        for (int r = 1; r < comm->world; ++r) acc += all[(size_t)r * d * d + e];
        mine[e] = acc;
      }
      NB_CUDA(cudaMemcpyAsync(cov.p, mine.data(), d * d * 8, cudaMemcpyHostToDevice, S));
    }
  }
  auto cov_apply = [&](const std::vector<double>& v, std::vector<double>& out) {
    NB_CUDA(cudaMemcpyAsync(vd.p, v.data(), d * 8, cudaMemcpyHostToDevice, S));
    if (fast) {
      k_cov_apply<<<(unsigned)((d * 32 + 255) / 256), 256, 0, S>>>(cov.p, vd.p, (uint32_t)d,
                                                                  1.0 / static_cast<double>(N), yd.p);
      note_launch(ctx, "k_cov_apply");
      out.resize(d);
      NB_CUDA(cudaMemcpyAsync(out.data(), yd.p, d * 8, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
      return;
    }
    auto cols = [&](int carry) {
      if (!n) return;
      k_pca_rows<<<row_blocks, 128, 0, S>>>(x, n, (uint32_t)d, mean.p, vd.p, t.p, nullptr,
                                            nullptr);
      note_launch(ctx, "k_pca_rows");
      k_pca_cols<BR><<<(unsigned)((d + 31) / 32), 256, col_smem, S>>>(x, n, (uint32_t)d, mean.p,
                                                                        t.p, yd.p, carry);
      note_launch(ctx, "k_pca_cols");
    };
    if (!comm) {
      cols(0);
    } else {  // y_j: the i-ascending chains continue rank to rank, then / N
      comm->chain(yd.p, d, [&] { cols(1); });
      k_div_vec<<<(unsigned)((d + 255) / 256), 256, 0, S>>>(yd.p, (uint32_t)d, (double)N);
      note_launch(ctx, "k_div_vec");
    }
    out.resize(d);
    NB_CUDA(cudaMemcpyAsync(out.data(), yd.p, d * 8, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
  };

  std::vector<double> applied(d);
  std::vector<std::vector<double>> basis(2, std::vector<double>(d));
  double eigen[2] = {0.0, 0.0};
  for (int comp = 0; comp < 2; ++comp) {  // pca.hpp:109-141
    std::vector<double>& v = basis[comp];
    for (double& e : v) e = rng.gaussian();
    if (comp == 1) {
      const double overlap = dot(v, basis[0]);
      for (uint64_t j = 0; j < d; ++j) v[j] -= overlap * basis[0][j];
    }
    if (normalize(v) == 0.0) continue;
    std::vector<double> prev(d);
    for (int iter = 0; iter < 3000; ++iter) {
      prev = v;
      cov_apply(v, applied);
      if (comp == 1) {
        const double overlap = dot(applied, basis[0]);
        for (uint64_t j = 0; j < d; ++j) applied[j] -= overlap * basis[0][j];
      }
      v = applied;
      if (normalize(v) == 0.0) {
        std::fill(v.begin(), v.end(), 0.0);
        break;
      }
      double drift = 0.0;
      const double align = dot(v, prev) < 0.0 ? -1.0 : 1.0;
      for (uint64_t j = 0; j < d; ++j) {
        const double diff = v[j] - align * prev[j];
        drift += diff * diff;
      }
      if (drift < 1e-30) break;
    }
    cov_apply(v, applied);
    eigen[comp] = dot(v, applied);
  }
  if (dot(basis[1], basis[1]) > 0.0) {  // pca.hpp:143-177
    const double overlap = dot(basis[1], basis[0]);
    for (uint64_t j = 0; j < d; ++j) basis[1][j] -= overlap * basis[0][j];
    if (normalize(basis[1]) > 0.0) {
      std::vector<double> ca, cb;
      cov_apply(basis[0], ca);
      cov_apply(basis[1], cb);
      const double h00 = dot(basis[0], ca), h01 = dot(basis[0], cb), h11 = dot(basis[1], cb);
      const double half_gap = 0.5 * (h00 - h11);
      const double root = std::sqrt(half_gap * half_gap + h01 * h01);
      eigen[0] = 0.5 * (h00 + h11) + root;
      eigen[1] = 0.5 * (h00 + h11) - root;
      double c = 1.0, s = 0.0;
      if (std::fabs(h01) > 1e-300) {
        const double tt = eigen[0] - h00;
        const double len = std::sqrt(h01 * h01 + tt * tt);
        c = h01 / len;
        s = tt / len;
      } else if (h11 > h00) {
        c = 0.0;
        s = 1.0;
      }
      std::vector<double> first(d), second(d);
      for (uint64_t j = 0; j < d; ++j) {
        first[j] = c * basis[0][j] + s * basis[1][j];
        second[j] = -s * basis[0][j] + c * basis[1][j];
      }
      basis[0] = first;
      basis[1] = second;
    }
  }
  for (auto& v : basis) {  // pca.hpp:179-187 sign rule
    uint64_t arg = 0;
    for (uint64_t j = 1; j < d; ++j)
      if (std::fabs(v[j]) > std::fabs(v[arg])) arg = j;
    if (v[arg] < 0.0)
      for (double& e : v) e = -e;
  }
  DBuf<double> b0(d), b1(d), st(2);
  NB_CUDA(cudaMemcpyAsync(b0.p, basis[0].data(), d * 8, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(b1.p, basis[1].data(), d * 8, cudaMemcpyHostToDevice, S));
  // layout_i[comp] = j-ascending chain (pca.hpp:199-204), both components in one pass
  if (n) {
    k_pca_rows<<<row_blocks, 128, 0, S>>>(x, n, (uint32_t)d, mean.p, b0.p, layout_out,
                                          layout_out + 1, b1.p);
    note_launch(ctx, "k_pca_rows");
  }
  const bool rank_deficient = eigen[1] <= 1e-12 * std::max(eigen[0], 0.0);
  for (int comp = 0; comp < 2; ++comp) {  // pca.hpp:189-216
    if (comp == 1 && rank_deficient) {
      if (n) {
        rng.g.discard(row0);  // the draws of the rows before this rank's
        std::vector<double> jit(n);
        for (uint64_t i = 0; i < n; ++i) jit[i] = -1e-4 + (1e-4 - -1e-4) * rng.uniform01();
        DBuf<double> jd(n);
        NB_CUDA(cudaMemcpyAsync(jd.p, jit.data(), n * 8, cudaMemcpyHostToDevice, S));
        k_layout_set<<<ctx->sm_count * 4, 256, 0, S>>>(layout_out, n, 1, jd.p);
        note_launch(ctx, "k_layout_set");
      }
      NB_CUDA(cudaStreamSynchronize(S));
      break;
    }
    // sequential column sums (pca.hpp:197-212), carried over the ranks
    auto col_sum = [&](int mode, double mu) {
      auto run = [&](int carry) {
        if (!n) return;
        k_seq_col<<<1, 256, 0, S>>>(layout_out, n, comp, mode, mu, st.p, carry);
        note_launch(ctx, "k_seq_col");
      };
      if (comm) comm->chain(st.p, 1, [&] { run(1); });
      else run(0);
      double h = 0.0;
      NB_CUDA(cudaMemcpyAsync(&h, st.p, 8, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
      return h;
    };
    const double col_mean = col_sum(0, 0.0) / static_cast<double>(N);
    const double sd = std::sqrt(col_sum(1, col_mean) / static_cast<double>(N));
    if (sd > 0.0 && n) {
      k_layout_scale<<<ctx->sm_count * 4, 256, 0, S>>>(layout_out, n, comp, sd);
      note_launch(ctx, "k_layout_scale");
    }
  }
  NB_CUDA(cudaStreamSynchronize(S));
}

}  // namespace nb

using namespace nb;

static int32_t pca_entry(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                         uint64_t seed, double* layout_out, int32_t location, bool fast) {
  return guard([&] {
    if (!ctx || !layout_out) fail(kParameter, "NULL argument");
    bind_device(ctx);
    DevData dd;
    dd.bind(data, ctx);
    if (location == NOMAD_B200_DEVICE) {
      pca_init_dev(ctx, dd.x, dd.n, dd.d, seed, layout_out, fast);
    } else {
      DBuf<double> lay(2 * dd.n);
      pca_init_dev(ctx, dd.x, dd.n, dd.d, seed, lay.p, fast);
      NB_CUDA(cudaMemcpy(layout_out, lay.p, dd.n * 16, cudaMemcpyDeviceToHost));
    }
  });
}

extern "C" int32_t nomad_b200_pca_init(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                       uint64_t seed, double* layout_out, int32_t location) {
  return pca_entry(ctx, data, seed, layout_out, location, false);
}

extern "C" int32_t nomad_b200_pca_init_fast(nomad_b200_ctx* ctx,
                                            const nomad_b200_dataset_view* data, uint64_t seed,
                                            double* layout_out, int32_t location) {
  return pca_entry(ctx, data, seed, layout_out, location, true);
}

// ---- row-sharded PCA: one rank's share of the rows
namespace nb {
static void pca_rank(nomad_b200_ctx* ctx, Comm* comm, const nomad_b200_dataset_view* rows,
                     uint64_t row0, uint64_t n_total, uint64_t seed, bool fast, double* layout_out,
                     int32_t location) {
  DevData dd;
  dd.bind(rows, ctx);
  if (row0 + dd.n > n_total) fail(kParameter, "row slice outside the dataset");
  if (location == NOMAD_B200_DEVICE) {
    pca_init_dev(ctx, dd.x, dd.n, dd.d, seed, layout_out, fast, comm, row0, n_total);
  } else {
    DBuf<double> lay(2 * dd.n);
    pca_init_dev(ctx, dd.x, dd.n, dd.d, seed, lay.p, fast, comm, row0, n_total);
    copy_d2h(ctx, layout_out, lay.p, dd.n * 16);
  }
}
}  // namespace nb

extern "C" int32_t nomad_b200_pca_init_sharded(nomad_b200_ctx* ctx, int32_t rank, int32_t world,
                                               const void* nccl_id,
                                               const nomad_b200_dataset_view* rows, uint64_t row0,
                                               uint64_t n_total, uint64_t seed, int32_t fast,
                                               double* layout_out, int32_t location) {
  return guard([&] {
    if (!ctx || !rows || !layout_out) fail(kParameter, "NULL argument");
    if (world < 1 || rank < 0 || rank >= world) fail(kParameter, "bad rank / world_size");
    bind_device(ctx);
    std::unique_ptr<Comm> comm(make_nccl_comm(rank, world, nccl_id, ctx->stream));
    pca_rank(ctx, comm.get(), rows, row0, n_total, seed, fast != 0, layout_out, location);
  });
}

extern "C" int32_t nomad_b200_group_pca_init_sharded(nomad_b200_group* grp,
                                                     const nomad_b200_dataset_view* rows,
                                                     const uint64_t* row0, uint64_t n_total,
                                                     uint64_t seed, int32_t fast,
                                                     double* const* layout_out, int32_t location) {
  return guard([&] {
    if (!grp || !rows || !row0 || !layout_out) fail(kParameter, "NULL argument");
    const int G = (int)grp->ctx.size();
    GroupRendezvous* rz = make_rendezvous(G);
    std::vector<std::exception_ptr> errs(G);
    std::vector<std::thread> th;
    for (int r = 0; r < G; ++r)
      th.emplace_back([&, r] {
        nomad_b200_ctx* c = grp->ctx[r];
        cudaStream_t shared = c->stream;
        cudaStream_t own = nullptr;
        try {
          bind_device(c);
          // a private stream per rank thread (loopback ranks share one)
          NB_CUDA(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
          c->stream = own;
          std::unique_ptr<Comm> comm(make_group_comm(rz, r, own, c->device));
          pca_rank(c, comm.get(), rows + r, row0[r], n_total, seed, fast != 0, layout_out[r],
                   location);
        } catch (...) {
          errs[r] = std::current_exception();
          rendezvous_abort(rz);
        }
        if (own) {
          cudaStreamSynchronize(own);
          cudaStreamDestroy(own);
        }
        c->stream = shared;
      });
    for (auto& t : th) t.join();
    free_rendezvous(rz);
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
  });
}

// Debug / unit path: covariance sums of a dataset about `mean` (host d
// doubles) into out (host d x d).
extern "C" int32_t nomad_b200_debug_cov(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                        const double* mean_host, double* out_host) {
  return guard([&] {
    if (!ctx || !mean_host || !out_host) fail(kParameter, "NULL argument");
    bind_device(ctx);
    DevData dd;
    dd.bind(data, ctx);
    DBuf<double> m(dd.d), c(dd.d * dd.d);
    NB_CUDA(cudaMemcpy(m.p, mean_host, dd.d * 8, cudaMemcpyHostToDevice));
    covariance_sums(ctx, dd.x, dd.n, dd.d, m.p, c.p);
    NB_CUDA(cudaMemcpy(out_host, c.p, dd.d * dd.d * 8, cudaMemcpyDeviceToHost));
  });
}
