// PCA initialisation (pca.hpp:79-218) on the GPU, tolerance parity: the two
// data passes of covariance_apply (pca.hpp:34-55) and the final projection
// run as fp64 kernels (tree reductions, so low-order bits differ from the
// reference's sequential sums); the d-dimensional vector algebra (deflation,
// normalisation, drift test, 2x2 Rayleigh-Ritz, sign rule) stays on the host
// in the reference's exact expression order, and the mean is the exact
// sequential mean. The start vectors and the rank-1 jitter come from the
// reference's own "pca" Rng stream.
#include <algorithm>
#include <cmath>

#include "index_common.cuh"

namespace nb {

namespace {

// t_i = sum_j (x_ij - mean_j) v_j   (warp per row)
__global__ void k_pca_rows(const float* __restrict__ x, uint64_t n, uint32_t d,
                           const double* __restrict__ mean, const double* __restrict__ v,
                           double* __restrict__ t) {
  const uint64_t row = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* xr = x + row * d;
  double acc = 0.0;
  for (uint32_t j = lane; j < d; j += 32) acc += ((double)xr[j] - mean[j]) * v[j];
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) t[row] = acc;
}

// y_j += sum_{i in chunk} (x_ij - mean_j) t_i   (block per row chunk,
// thread per column, one atomic per (block, column))
__global__ void k_pca_cols(const float* __restrict__ x, uint64_t n, uint32_t d,
                           const double* __restrict__ mean, const double* __restrict__ t,
                           uint64_t rows_per_block, double* __restrict__ y) {
  const uint64_t r0 = blockIdx.x * rows_per_block;
  const uint64_t r1 = umin64(r0 + rows_per_block, n);
  for (uint32_t j = threadIdx.x; j < d; j += blockDim.x) {
    double acc = 0.0;
    const double m = mean[j];
    for (uint64_t i = r0; i < r1; ++i) acc += ((double)x[i * d + j] - m) * t[i];
    atomicAdd(&y[j], acc);
  }
}

// layout_i = (sum_j (x_ij - mean_j) b0_j, sum_j (x_ij - mean_j) b1_j)
__global__ void k_pca_project(const float* __restrict__ x, uint64_t n, uint32_t d,
                              const double* __restrict__ mean, const double* __restrict__ b0,
                              const double* __restrict__ b1, double* __restrict__ out) {
  const uint64_t row = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* xr = x + row * d;
  double a0 = 0.0, a1 = 0.0;
  for (uint32_t j = lane; j < d; j += 32) {
    const double c = (double)xr[j] - mean[j];
    a0 += c * b0[j];
    a1 += c * b1[j];
  }
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
  }
  if (lane == 0) {
    out[2 * row] = a0;
    out[2 * row + 1] = a1;
  }
}

// sums of (x - mean)^2 and x^2 over all entries; column sums / sq of layout
__global__ void k_pca_moments(const float* __restrict__ x, uint64_t N, uint32_t d,
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

__global__ void k_layout_stats(const double* lay, uint64_t n, int comp, double mu, double* out) {
  double s = 0.0, q = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double v = lay[2 * i + comp];
    s += v;
    const double c = v - mu;
    q += c * c;
  }
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    q += __shfl_xor_sync(0xffffffffu, q, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], s);
    atomicAdd(&out[1], q);
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

// layout_out: device n x 2.
void pca_init_dev(nomad_b200_ctx* ctx, const float* x, uint64_t n, uint64_t d, uint64_t seed,
                  double* layout_out) {
  cudaStream_t S = ctx->stream;
  if (n < 2) fail(kParameter, "need at least 2 rows");
  HostRng rng(HostRng::stream_seed(seed, 0x706361 /* "pca" */));
  DBuf<double> mean(d), vd(d), yd(d), t(n), mom(2);
  seq_column_means(ctx, x, d, nullptr, {0}, {n}, {0}, mean.p);  // pca.hpp:84-89
  NB_CUDA(cudaMemsetAsync(mom.p, 0, 16, S));
  k_pca_moments<<<ctx->sm_count * 8, 256, 0, S>>>(x, n * d, (uint32_t)d, mean.p, mom.p);
  note_launch(ctx, "k_pca_moments");
  double mh[2];
  NB_CUDA(cudaMemcpyAsync(mh, mom.p, 16, cudaMemcpyDeviceToHost, S));
  NB_CUDA(cudaStreamSynchronize(S));
  const double total_var = mh[0] / static_cast<double>(n);
  const double total_sq = mh[1] / static_cast<double>(n);
  if (total_var <= 1e-18 * std::max(1.0, total_sq))
    fail(kDegenerate, "data has zero variance");

  const unsigned rows_blocks = (unsigned)((n * 32 + 255) / 256);
  const uint64_t rpb = std::max<uint64_t>(64, (n + ctx->sm_count * 16 - 1) / (ctx->sm_count * 16));
  const unsigned col_blocks = (unsigned)((n + rpb - 1) / rpb);
  auto cov_apply = [&](const std::vector<double>& v, std::vector<double>& out) {
    NB_CUDA(cudaMemcpyAsync(vd.p, v.data(), d * 8, cudaMemcpyHostToDevice, S));
    k_pca_rows<<<rows_blocks, 256, 0, S>>>(x, n, (uint32_t)d, mean.p, vd.p, t.p);
    note_launch(ctx, "k_pca_rows");
    NB_CUDA(cudaMemsetAsync(yd.p, 0, d * 8, S));
    k_pca_cols<<<col_blocks, std::min<unsigned>(256, ((unsigned)d + 31) / 32 * 32), 0, S>>>(
        x, n, (uint32_t)d, mean.p, t.p, rpb, yd.p);
    note_launch(ctx, "k_pca_cols");
    out.resize(d);
    NB_CUDA(cudaMemcpyAsync(out.data(), yd.p, d * 8, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    for (double& o : out) o /= static_cast<double>(n);
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
  k_pca_project<<<rows_blocks, 256, 0, S>>>(x, n, (uint32_t)d, mean.p, b0.p, b1.p, layout_out);
  note_launch(ctx, "k_pca_project");
  const bool rank_deficient = eigen[1] <= 1e-12 * std::max(eigen[0], 0.0);
  for (int comp = 0; comp < 2; ++comp) {  // pca.hpp:189-216
    if (comp == 1 && rank_deficient) {
      std::vector<double> jit(n);
      for (uint64_t i = 0; i < n; ++i) jit[i] = -1e-4 + (1e-4 - -1e-4) * rng.uniform01();
      DBuf<double> jd(n);
      NB_CUDA(cudaMemcpyAsync(jd.p, jit.data(), n * 8, cudaMemcpyHostToDevice, S));
      k_layout_set<<<ctx->sm_count * 4, 256, 0, S>>>(layout_out, n, 1, jd.p);
      note_launch(ctx, "k_layout_set");
      NB_CUDA(cudaStreamSynchronize(S));
      break;
    }
    double h[2];
    NB_CUDA(cudaMemsetAsync(st.p, 0, 16, S));
    k_layout_stats<<<ctx->sm_count * 4, 256, 0, S>>>(layout_out, n, comp, 0.0, st.p);
    NB_CUDA(cudaMemcpyAsync(h, st.p, 16, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    const double col_mean = h[0] / static_cast<double>(n);
    NB_CUDA(cudaMemsetAsync(st.p, 0, 16, S));
    k_layout_stats<<<ctx->sm_count * 4, 256, 0, S>>>(layout_out, n, comp, col_mean, st.p);
    note_launch(ctx, "k_layout_stats");
    NB_CUDA(cudaMemcpyAsync(h, st.p, 16, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    const double sd = std::sqrt(h[1] / static_cast<double>(n));
    if (sd > 0.0) {
      k_layout_scale<<<ctx->sm_count * 4, 256, 0, S>>>(layout_out, n, comp, sd);
      note_launch(ctx, "k_layout_scale");
    }
  }
  NB_CUDA(cudaStreamSynchronize(S));
}

}  // namespace nb

using namespace nb;

extern "C" int32_t nomad_b200_pca_init(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                       uint64_t seed, double* layout_out, int32_t location) {
  return guard([&] {
    if (!ctx || !layout_out) fail(kParameter, "NULL argument");
    bind_device(ctx);
    DevData dd;
    dd.bind(data, ctx->stream);
    if (location == NOMAD_B200_DEVICE) {
      pca_init_dev(ctx, dd.x, dd.n, dd.d, seed, layout_out);
    } else {
      DBuf<double> lay(2 * dd.n);
      pca_init_dev(ctx, dd.x, dd.n, dd.d, seed, lay.p);
      NB_CUDA(cudaMemcpy(layout_out, lay.p, dd.n * 16, cudaMemcpyDeviceToHost));
    }
  });
}
