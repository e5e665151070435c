// K1-K5: the LSH-seeded Lloyd k-means partitioner (kmeans.hpp:47-296) on the
// GPU, exact: every distance is the reference's j-ascending fp64 chain with
// no FMA (_rn intrinsics), argmins keep the lowest index on ties, and every
// centroid / mean is a sequential sum in ascending point id, so assignments,
// centroids, sizes and the quantisation-error trace are bit-identical to the
// reference. Host work is limited to O(C), O(2^planes) and O(planes * d)
// bookkeeping (bucket ranking, the Rng draws, stop rule).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "index_common.cuh"
#include "shard.cuh"

namespace nb {

namespace {

// ------------------------------------------------------------ K3 assign
//
// Block tile = (16 * PPT) points x (16 * CPT) centroids; thread (tx, ty)
// owns points ty + 16 i and centroids tx + 16 c of the tile (strided, so the
// shared-memory reads are conflict-free), with PPT * CPT = 16 independent
// distance chains. Centroid tiles are visited in ascending order and each
// thread keeps its running (best, index) with a strict '<'; the 16 threads
// sharing a point then combine by (distance, index) — which reproduces
// nearest_centroid's first-minimum scan (kmeans.hpp:56-68).
template <int PPT, int CPT>
__global__ void __launch_bounds__(256) k_assign(XPtr x, uint64_t n,
                                                uint32_t d, const double* __restrict__ cent,
                                                uint32_t C, uint32_t* assign,
                                                unsigned long long* changes, int count_changes) {
  constexpr int TP = 16 * PPT, TC = 16 * CPT, DK = 32;
  // dynamic: xs[TP][DK+1] doubles, cs[TC][DK+1] doubles, xf[TP*DK] f32 (the
  // next x tile in flight by cp.async while the current one is consumed;
  // each thread widens exactly the elements it copied)
  extern __shared__ __align__(16) double kasm[];
  double (*xs)[DK + 1] = reinterpret_cast<double (*)[DK + 1]>(kasm);
  double (*cs)[DK + 1] = reinterpret_cast<double (*)[DK + 1]>(kasm + TP * (DK + 1));
  float* xf = reinterpret_cast<float*>(kasm + (TP + TC) * (DK + 1));
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const uint64_t p0 = (uint64_t)blockIdx.x * TP;
  double best[PPT];
  uint32_t bidx[PPT];
#pragma unroll
  for (int i = 0; i < PPT; ++i) {
    best[i] = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    bidx[i] = 0;
  }
  for (uint32_t c0 = 0; c0 < C; c0 += TC) {
    double acc[PPT][CPT];
#pragma unroll
    for (int i = 0; i < PPT; ++i)
#pragma unroll
      for (int c = 0; c < CPT; ++c) acc[i][c] = 0.0;
    // x tile j0 -> xf (f32 rows: cp.async; bf16 rows: widened plain loads)
    auto stage_x = [&](uint32_t j0) {
      for (int e = threadIdx.x; e < TP * DK; e += 256) {
        const int p = e / DK, jj = e % DK;
        const uint64_t gp = p0 + p;
        const uint32_t j = j0 + jj;
        if (gp < n && j < d) {
          if (x.bf) {
            xf[e] = x[gp * d + j];
          } else {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(xf + e)),
                         "l"(static_cast<const float*>(x.p) + gp * d + j)
                         : "memory");
          }
        } else {
          xf[e] = 0.f;
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    stage_x(0);
    for (uint32_t j0 = 0; j0 < d; j0 += DK) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      for (int e = threadIdx.x; e < TP * DK; e += 256) xs[e / DK][e % DK] = (double)xf[e];
      for (int e = threadIdx.x; e < TC * DK; e += 256) {
        const int r = e / DK, jj = e % DK;
        const uint32_t gr = c0 + r, j = j0 + jj;
        cs[r][jj] = (gr < C && j < d) ? cent[(uint64_t)gr * d + j] : 0.0;
      }
      __syncthreads();
      if (j0 + DK < d) stage_x(j0 + DK);  // own elements only: already widened
      const int jmax = min(DK, (int)(d - j0));
      for (int jj = 0; jj < jmax; ++jj) {
        double xv[PPT], cv[CPT];
#pragma unroll
        for (int i = 0; i < PPT; ++i) xv[i] = xs[ty + 16 * i][jj];
#pragma unroll
        for (int c = 0; c < CPT; ++c) cv[c] = cs[tx + 16 * c][jj];
#pragma unroll
        for (int i = 0; i < PPT; ++i)
#pragma unroll
          for (int c = 0; c < CPT; ++c) {
            const double diff = __dsub_rn(xv[i], cv[c]);
            acc[i][c] = __dadd_rn(acc[i][c], __dmul_rn(diff, diff));
          }
      }
      __syncthreads();  // xs / cs are rewritten by the next step
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const uint32_t r = c0 + tx + 16 * c;
      if (r < C) {
#pragma unroll
        for (int i = 0; i < PPT; ++i)
          if (acc[i][c] < best[i]) {
            best[i] = acc[i][c];
            bidx[i] = r;
          }
      }
    }
  }
  // combine the 16 threads of a point (lanes tx = 0..15 of a half warp)
  unsigned long long ch = 0;
#pragma unroll
  for (int i = 0; i < PPT; ++i) {
    double b = best[i];
    uint32_t bi = bidx[i];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, b, o);
      const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob < b || (ob == b && oi < bi)) {
        b = ob;
        bi = oi;
      }
    }
    const uint64_t gp = p0 + ty + 16 * i;
    if (tx == 0 && gp < n) {
      if (count_changes && assign[gp] != bi) ++ch;
      assign[gp] = bi;
    }
  }
  if (count_changes) {
    for (int o = 16; o > 0; o >>= 1) ch += __shfl_xor_sync(0xffffffffu, ch, o);
    if ((threadIdx.x & 31) == 0 && ch) atomicAdd(changes, ch);
  }
}

// Rows of x staged through shared memory (coalesced), then one thread per
// point runs its j-ascending fp64 chain: sq_dist (kmeans.hpp:47-54) to the
// centroid `cent + cidx[i] * d` (cidx == nullptr: the single row `cent`).
__global__ void __launch_bounds__(128) k_point_sqdist(XPtr x, uint64_t n,
                                                      uint32_t d, const double* __restrict__ cent,
                                                      const uint32_t* cidx, double* out) {
  constexpr int TP = 128, DK = 32;
  __shared__ float xs[TP][DK + 1];
  const uint64_t p0 = (uint64_t)blockIdx.x * TP;
  const uint64_t gp = p0 + threadIdx.x;
  const double* c = cent + (cidx && gp < n ? (uint64_t)cidx[gp] * d : 0);
  double acc = 0.0;
  for (uint32_t j0 = 0; j0 < d; j0 += DK) {
    __syncthreads();
    for (int e = threadIdx.x; e < TP * DK; e += TP) {
      const int p = e / DK, jj = e % DK;
      const uint64_t q = p0 + p;
      xs[p][jj] = (q < n && j0 + jj < d) ? x[q * d + j0 + jj] : 0.f;
    }
    __syncthreads();
    const int jmax = min(DK, (int)(d - j0));
    for (int jj = 0; jj < jmax; ++jj) {
      const double diff = __dsub_rn((double)xs[threadIdx.x][jj], c[j0 + jj]);
      acc = __dadd_rn(acc, __dmul_rn(diff, diff));
    }
  }
  if (gp < n) out[gp] = acc;
}

// K1: LSH codes (kmeans.hpp:188-201). One thread per point; for each j the
// centred value ((double)x_j - mean_j) feeds all planes' j-ascending chains.
__global__ void __launch_bounds__(128) k_lsh_hash(XPtr x, uint64_t n,
                                                  uint32_t d, const double* __restrict__ mean,
                                                  const double* __restrict__ planes, uint32_t P,
                                                  uint32_t* codes) {
  constexpr int TP = 128, DK = 32, PMAX = 24;
  __shared__ float xs[TP][DK + 1];
  __shared__ double ms[DK];
  __shared__ double ws[PMAX][DK];
  const uint64_t p0 = (uint64_t)blockIdx.x * TP;
  const uint64_t gp = p0 + threadIdx.x;
  double proj[PMAX];
#pragma unroll
  for (int p = 0; p < PMAX; ++p) proj[p] = 0.0;
  for (uint32_t j0 = 0; j0 < d; j0 += DK) {
    __syncthreads();
    for (int e = threadIdx.x; e < TP * DK; e += TP) {
      const int p = e / DK, jj = e % DK;
      const uint64_t q = p0 + p;
      xs[p][jj] = (q < n && j0 + jj < d) ? x[q * d + j0 + jj] : 0.f;
    }
    for (int e = threadIdx.x; e < DK; e += TP) ms[e] = j0 + e < d ? mean[j0 + e] : 0.0;
    for (int e = threadIdx.x; e < (int)P * DK; e += TP) {
      const int p = e / DK, jj = e % DK;
      ws[p][jj] = j0 + jj < d ? planes[(uint64_t)p * d + j0 + jj] : 0.0;
    }
    __syncthreads();
    const int jmax = min(DK, (int)(d - j0));
    for (int jj = 0; jj < jmax; ++jj) {
      const double c = __dsub_rn((double)xs[threadIdx.x][jj], ms[jj]);
#pragma unroll
      for (int p = 0; p < PMAX; ++p)
        if (p < (int)P) proj[p] = __dadd_rn(proj[p], __dmul_rn(c, ws[p][jj]));
    }
  }
  if (gp < n) {
    uint32_t code = 0;
#pragma unroll
    for (int p = 0; p < PMAX; ++p)
      if (p < (int)P && proj[p] >= 0.0) code |= 1u << p;
    codes[gp] = code;
  }
}

__global__ void k_sizes(const uint32_t* a, uint64_t n, uint32_t* sizes) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    atomicAdd(&sizes[a[i]], 1u);
}

// Sequential fp64 sum of v[0..n) in order (one thread adds; the block stages
// the next tile into shared memory). Used where the reference accumulates a
// scalar over points in order (quantization_error, the perturbation scale).
__global__ void k_seq_sum(const double* v, uint64_t n, double* out, int carry) {
  constexpr int T = 2048;
  __shared__ double buf[2][T];
  double acc = carry ? *out : 0.0;  // carry: continue the previous rank's running sum
  int cur = 0;
  for (uint64_t e = threadIdx.x; e < T && e < n; e += blockDim.x) buf[0][e] = v[e];
  __syncthreads();
  for (uint64_t b = 0; b < n; b += T) {
    const uint64_t nb = b + T;
    for (uint64_t e = threadIdx.x; e < T && nb + e < n; e += blockDim.x) buf[cur ^ 1][e] = v[nb + e];
    if (threadIdx.x == 0) {
      const uint64_t m = umin64(T, n - b);
      for (uint64_t e = 0; e < m; ++e) acc = __dadd_rn(acc, buf[cur][e]);
    }
    __syncthreads();
    cur ^= 1;
  }
  if (threadIdx.x == 0) *out = acc;
}

// default_kmeans_tol accumulator (kmeans.hpp:157-161): storage-order
// sequential sum of the exact products (double)v * v.
__global__ void k_seq_sumsq(XPtr v, uint64_t n, double* out, int carry) {
  constexpr int T = 4096;
  __shared__ float buf[2][T];
  double acc = carry ? *out : 0.0;
  int cur = 0;
  for (uint64_t e = threadIdx.x; e < T && e < n; e += blockDim.x) buf[0][e] = v[e];
  __syncthreads();
  for (uint64_t b = 0; b < n; b += T) {
    const uint64_t nb = b + T;
    for (uint64_t e = threadIdx.x; e < T && nb + e < n; e += blockDim.x) buf[cur ^ 1][e] = v[nb + e];
    if (threadIdx.x == 0) {
      const uint64_t m = umin64(T, n - b);
      for (uint64_t e = 0; e < m; ++e) {
        const double w = (double)buf[cur][e];
        acc = __dadd_rn(acc, __dmul_rn(w, w));
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  if (threadIdx.x == 0) *out = acc;
}

// Any-order parallel sum of the same exact products (for the tolerance
// bracket); partial per block.
__global__ void k_par_sumsq(XPtr v, uint64_t n, double* part) {
  __shared__ double red[32];
  double acc = 0.0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const double w = (double)v[i];
    acc = __dadd_rn(acc, __dmul_rn(w, w));
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    part[blockIdx.x] = s;
  }
}

// kmeans.hpp:282-290 per-cluster squared move, j-ascending.
__global__ void k_moves(const double* cnew, const double* cold, uint32_t C, uint32_t d,
                        double* out) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= C) return;
  double mv = 0.0;
  for (uint32_t j = 0; j < d; ++j) {
    const double diff = __dsub_rn(cnew[(uint64_t)r * d + j], cold[(uint64_t)r * d + j]);
    mv = __dadd_rn(mv, __dmul_rn(diff, diff));
  }
  out[r] = mv;
}

// repair: farthest point of `donor` (max distance, then lowest id).
__global__ void k_far_max(const double* dist, const uint32_t* a, uint64_t n, uint32_t donor,
                          unsigned long long* best_bits) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (a[i] == donor) atomicMax(best_bits, (unsigned long long)__double_as_longlong(dist[i]));
}
__global__ void k_far_argmin(const double* dist, const uint32_t* a, uint64_t n, uint32_t donor,
                             const unsigned long long* best_bits, unsigned long long* idx) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (a[i] == donor && (unsigned long long)__double_as_longlong(dist[i]) == *best_bits)
      atomicMin(idx, (unsigned long long)i);
}
__global__ void k_set_u32(uint32_t* p, uint64_t i, uint32_t v) { p[i] = v; }

// rows r of `m` (rows x d sums) with div[r] > 0 divided by div[r] (the carry
// chain's final step: kmeans.hpp:98-103 skips empty clusters)
__global__ void k_div_rows(double* m, uint32_t rows, uint32_t d, const double* div) {
  const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (e >= (uint64_t)rows * d) return;
  const double v = div[e / d];
  if (v > 0.0) m[e] = __ddiv_rn(m[e], v);
}

unsigned grid_for(uint64_t n, unsigned t, unsigned cap) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(cap, (n + t - 1) / t));
}

}  // namespace

// --------------------------------------------------------------- host side

struct KMeans {
  nomad_b200_ctx* ctx;
  XPtr x;
  uint64_t n, d;  // this rank's rows (all rows on one GPU)
  uint32_t C;
  // row-sharded build (shard.cuh): rows [row0, row0 + n) of n_total
  Comm* comm = nullptr;
  uint64_t row0 = 0, n_total = 0;
  DBuf<uint32_t> a;        // assignment
  DBuf<double> cent;       // C x d
  DBuf<uint32_t> sizes_d;  // C
  std::vector<uint32_t> sizes;
  DBuf<double> dist;       // n (scratch)
  DBuf<double> scal;       // scratch scalars
  DBuf<unsigned long long> u64s;

  KMeans(nomad_b200_ctx* c, XPtr xx, uint64_t nn, uint64_t dd, uint32_t CC)
      : ctx(c), x(xx), n(nn), d(dd), C(CC), n_total(nn) {
    a.alloc(n);
    cent.alloc((uint64_t)C * d);
    sizes_d.alloc(C);
    scal.alloc(4);
    u64s.alloc(4);
  }
  cudaStream_t S() const { return ctx->stream; }

  void assign(bool count, unsigned long long* changes_out) {
    NB_CUDA(cudaMemsetAsync(u64s.p, 0, 8, S()));
    if (!n) {  // a rank without rows still takes part in the count
      if (changes_out) {
        *changes_out = 0;
        if (comm) {
          uint64_t c = 0;
          comm->allreduce_u64(&c, 1);
          *changes_out = c;
        }
      }
      return;
    }
    auto go = [&](auto kern, int tp, int tc) {
      const size_t smem = (size_t)(tp + tc) * 33 * 8 + (size_t)tp * 32 * 4;
      NB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<(unsigned)((n + tp - 1) / tp), 256, smem, S()>>>(x, n, (uint32_t)d, cent.p, C, a.p,
                                                              u64s.p, count ? 1 : 0);
    };
    if (C > 32) go(k_assign<4, 4>, 64, 64);
    else if (C > 16) go(k_assign<8, 2>, 128, 32);
    else go(k_assign<8, 1>, 128, 16);
    note_launch(ctx, "k_assign");
    if (changes_out) {
      NB_CUDA(cudaMemcpyAsync(changes_out, u64s.p, 8, cudaMemcpyDeviceToHost, S()));
      NB_CUDA(cudaStreamSynchronize(S()));
      if (comm) {
        uint64_t c = *changes_out;
        comm->allreduce_u64(&c, 1);
        *changes_out = c;
      }
    }
  }

  // Sequential ascending-id column sums over segments of this rank's rows
  // (members: local row indices), divided by the global counts `div` — on
  // one GPU seq_column_means itself; row-sharded, the carry chain.
  void seq_means(const uint32_t* members, const std::vector<uint64_t>& beg,
                 const std::vector<uint64_t>& cnt, const std::vector<uint32_t>& rows,
                 const std::vector<double>& div, double* out, uint32_t out_rows) {
    if (!comm) {
      seq_column_means(ctx, x, d, members, beg, cnt, rows, out);
      return;
    }
    comm->chain(out, (size_t)out_rows * d, [&] {
      seq_column_means(ctx, x, d, members, beg, cnt, rows, out, true);
    });
    DBuf<double> dv(out_rows);
    NB_CUDA(cudaMemcpyAsync(dv.p, div.data(), out_rows * 8, cudaMemcpyHostToDevice, S()));
    const uint64_t e = (uint64_t)out_rows * d;
    k_div_rows<<<(unsigned)((e + 255) / 256), 256, 0, S()>>>(out, out_rows, (uint32_t)d, dv.p);
    note_launch(ctx, "k_div_rows");
    NB_CUDA(cudaStreamSynchronize(S()));
  }
  // Sequential sum of v[0..n) (kmeans.hpp:148-154, :228-231): a carry chain
  // when row-sharded.
  double seq_sum(const double* v) {
    auto run = [&](int carry) {
      k_seq_sum<<<1, 256, 0, S()>>>(v, n, scal.p, carry);
      note_launch(ctx, "k_seq_sum");
    };
    if (comm) comm->chain(scal.p, 1, [&] { run(1); });
    else run(0);
    double acc = 0.0;
    NB_CUDA(cudaMemcpyAsync(&acc, scal.p, 8, cudaMemcpyDeviceToHost, S()));
    NB_CUDA(cudaStreamSynchronize(S()));
    return acc;
  }

  void recompute_sizes() {
    NB_CUDA(cudaMemsetAsync(sizes_d.p, 0, C * 4, S()));
    k_sizes<<<grid_for(n, 256, 4096), 256, 0, S()>>>(a.p, n, sizes_d.p);
    note_launch(ctx, "k_sizes");
    sizes.resize(C);
    NB_CUDA(cudaMemcpyAsync(sizes.data(), sizes_d.p, C * 4, cudaMemcpyDeviceToHost, S()));
    NB_CUDA(cudaStreamSynchronize(S()));
    if (comm) {  // global sizes on every rank
      std::vector<uint64_t> g(sizes.begin(), sizes.end());
      comm->allreduce_u64(g.data(), C);
      for (uint32_t r = 0; r < C; ++r) sizes[r] = (uint32_t)g[r];
      NB_CUDA(cudaMemcpyAsync(sizes_d.p, sizes.data(), C * 4, cudaMemcpyHostToDevice, S()));
      NB_CUDA(cudaStreamSynchronize(S()));
    }
  }

  // kmeans.hpp:90-104: zero every centroid, sum members ascending, divide
  // the non-empty ones.
  void recompute_all() {
    NB_CUDA(cudaMemsetAsync(cent.p, 0, (uint64_t)C * d * 8, S()));
    DBuf<uint32_t> mem;
    std::vector<uint64_t> off;
    group_by_label(ctx, a.p, n, C, mem, off);
    std::vector<uint64_t> beg, cnt;
    std::vector<uint32_t> rows;
    std::vector<double> div(C, 0.0);
    for (uint32_t r = 0; r < C; ++r) {
      div[r] = (double)sizes[r];
      if (off[r + 1] > off[r]) {
        beg.push_back(off[r]);
        cnt.push_back(off[r + 1] - off[r]);
        rows.push_back(r);
      }
    }
    seq_means(mem.p, beg, cnt, rows, div, cent.p, C);
  }

  // kmeans.hpp:75-88 for one cluster (members ascending; zero if empty).
  void recompute_one(uint32_t r) {
    NB_CUDA(cudaMemsetAsync(cent.p + (uint64_t)r * d, 0, d * 8, S()));
    // members of r only: labels == r, everything else dropped
    DBuf<uint32_t> lab(n);
    // map a -> (a == r ? 0 : 1) with L = 1
    map_eq(r, lab.p);
    DBuf<uint32_t> mem;
    std::vector<uint64_t> off;
    group_by_label(ctx, lab.p, n, 1, mem, off);
    if (!comm) {
      if (off[1] > 0) seq_column_means(ctx, x, d, mem.p, {0}, {off[1]}, {r}, cent.p);
      return;
    }
    // row-sharded: chain over the one row, then / its global size
    DBuf<double> row(d);
    std::vector<uint64_t> b, c;
    std::vector<uint32_t> rr;
    if (off[1] > 0) {
      b.push_back(0);
      c.push_back(off[1]);
      rr.push_back(0);
    }
    seq_means(mem.p, b, c, rr, {(double)sizes[r]}, row.p, 1);
    NB_CUDA(cudaMemcpyAsync(cent.p + (uint64_t)r * d, row.p, d * 8, cudaMemcpyDeviceToDevice, S()));
    NB_CUDA(cudaStreamSynchronize(S()));
  }

  void map_eq(uint32_t r, uint32_t* out);

  // kmeans.hpp:109-143
  void repair() {
    for (;;) {
      uint32_t empty = 0xFFFFFFFFu;
      for (uint32_t r = 0; r < C; ++r)
        if (sizes[r] == 0) { empty = r; break; }
      if (empty == 0xFFFFFFFFu) return;
      uint32_t donor = 0;
      for (uint32_t r = 1; r < C; ++r)
        if (sizes[r] > sizes[donor]) donor = r;
      if (sizes[donor] < 2) fail(kInternal, "no donor cluster available for repair");
      dist.alloc(n);
      DBuf<uint32_t> cidx(1);
      // distances of every point to the donor centroid (only donor's used)
      k_point_sqdist<<<(unsigned)((n + 127) / 128), 128, 0, S()>>>(
          x, n, (uint32_t)d, cent.p + (uint64_t)donor * d, nullptr, dist.p);
      note_launch(ctx, "k_point_sqdist");
      NB_CUDA(cudaMemsetAsync(u64s.p, 0, 8, S()));
      NB_CUDA(cudaMemsetAsync(u64s.p + 1, 0xFF, 8, S()));
      k_far_max<<<grid_for(n, 256, 4096), 256, 0, S()>>>(dist.p, a.p, n, donor, u64s.p);
      k_far_argmin<<<grid_for(n, 256, 4096), 256, 0, S()>>>(dist.p, a.p, n, donor, u64s.p,
                                                            u64s.p + 1);
      note_launch(ctx, "k_far_argmin");
      unsigned long long best[2] = {0, 0};  // distance bits (0: none), local index
      NB_CUDA(cudaMemcpyAsync(best, u64s.p, 16, cudaMemcpyDeviceToHost, S()));
      NB_CUDA(cudaStreamSynchronize(S()));
      unsigned long long victim = best[1];
      bool mine = true;
      if (comm) {  // the farthest over all ranks (larger distance, then lower id)
        unsigned long long cand[2] = {best[0], best[1] == ~0ull ? ~0ull : row0 + best[1]};
        std::vector<unsigned long long> all(2 * (size_t)comm->world);
        comm->allgather(cand, 16, all.data());
        int win = -1;
        for (int rk = 0; rk < comm->world; ++rk) {
          const unsigned long long b = all[2 * rk], id = all[2 * rk + 1];
          if (id == ~0ull) continue;
          if (win < 0 || b > all[2 * win] || (b == all[2 * win] && id < all[2 * win + 1])) win = rk;
        }
        mine = win == comm->rank;
        victim = best[1];
      }
      if (mine) {
        k_set_u32<<<1, 1, 0, S()>>>(a.p, victim, empty);
        note_launch(ctx, "k_set_u32");
      }
      --sizes[donor];
      ++sizes[empty];
      NB_CUDA(cudaMemcpyAsync(sizes_d.p, sizes.data(), C * 4, cudaMemcpyHostToDevice, S()));
      recompute_one(donor);
      recompute_one(empty);
    }
  }

  double quantization_error() {  // kmeans.hpp:148-154
    dist.alloc(std::max<uint64_t>(n, 1));
    if (n) {
      k_point_sqdist<<<(unsigned)((n + 127) / 128), 128, 0, S()>>>(x, n, (uint32_t)d, cent.p,
                                                                  a.p, dist.p);
      note_launch(ctx, "k_point_sqdist");
    }
    return seq_sum(dist.p) / static_cast<double>(n_total);
  }
};

namespace {
__global__ void k_map_eq(const uint32_t* a, uint64_t n, uint32_t r, uint32_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = a[i] == r ? 0u : 1u;
}
}  // namespace

void KMeans::map_eq(uint32_t r, uint32_t* out) {
  k_map_eq<<<grid_for(n, 256, 4096), 256, 0, S()>>>(a.p, n, r, out);
  note_launch(ctx, "k_map_eq");
}

// Exact default_kmeans_tol (kmeans.hpp:157-161): one sequential chain (a
// carry chain over the ranks when row-sharded).
double default_tol_exact(nomad_b200_ctx* ctx, XPtr x, uint64_t n, uint64_t d,
                         Comm* comm = nullptr, uint64_t n_total = 0) {
  DBuf<double> o(1);
  auto run = [&](int carry) {
    k_seq_sumsq<<<1, 1024, 0, ctx->stream>>>(x, n * d, o.p, carry);
    note_launch(ctx, "k_seq_sumsq");
  };
  if (comm) comm->chain(o.p, 1, [&] { run(1); });
  else run(0);
  double acc = 0.0;
  NB_CUDA(cudaMemcpyAsync(&acc, o.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  NB_CUDA(cudaStreamSynchronize(ctx->stream));
  return 1e-6 * (acc / static_cast<double>(comm ? n_total : n));
}

// [lo, hi] bracket of default_kmeans_tol from an any-order parallel sum:
// for N non-negative terms any summation order is within (N-1)u of the
// exact sum, so the sequential result lies within a factor (1 +- g)^2.
void default_tol_bracket(nomad_b200_ctx* ctx, XPtr x, uint64_t n, uint64_t d,
                         double* lo, double* hi, Comm* comm = nullptr, uint64_t n_total = 0) {
  const uint64_t N = n * d;
  const unsigned blocks = grid_for(std::max<uint64_t>(N, 1), 256, 2048);
  DBuf<double> part(blocks);
  NB_CUDA(cudaMemsetAsync(part.p, 0, blocks * 8, ctx->stream));
  if (N) {
    k_par_sumsq<<<blocks, 256, 0, ctx->stream>>>(x, N, part.p);
    note_launch(ctx, "k_par_sumsq");
  }
  std::vector<double> h(blocks);
  NB_CUDA(cudaMemcpyAsync(h.data(), part.p, blocks * 8, cudaMemcpyDeviceToHost, ctx->stream));
  NB_CUDA(cudaStreamSynchronize(ctx->stream));
  double s = 0.0;
  for (double v : h) s += v;
  uint64_t NT = N + blocks, nn = n;
  if (comm) {  // any order of any partial sums stays inside the bracket
    std::vector<double> all(comm->world);
    comm->allgather(&s, 8, all.data());
    s = 0.0;
    for (double v : all) s += v;
    NT = n_total * d + (uint64_t)blocks * comm->world + comm->world;
    nn = n_total;
  }
  const double u = 0x1p-53;
  const double g = (double)NT * u * 1.0001;
  const double slo = s * (1.0 - g) * (1.0 - g), shi = s * (1.0 + g) * (1.0 + g);
  *lo = 1e-6 * (std::nextafter(slo, 0.0) / static_cast<double>(nn));
  *hi = 1e-6 * (std::nextafter(shi, INFINITY) / static_cast<double>(nn));
}

// kmeans.hpp:167-250
void lsh_init_dev(nomad_b200_ctx* ctx, KMeans& km, uint64_t seed) {
  const uint64_t n = km.n, d = km.d;
  const uint32_t C = km.C;
  cudaStream_t S = ctx->stream;
  HostRng rng(HostRng::stream_seed(seed, 0x6c7368 /* "lsh" */));
  // data mean, ascending i (kmeans.hpp:176-181)
  DBuf<double> mean(d);
  {
    std::vector<uint64_t> b, c;
    std::vector<uint32_t> r;
    if (n) {
      b.push_back(0);
      c.push_back(n);
      r.push_back(0);
    }
    km.seq_means(nullptr, b, c, r, {(double)km.n_total}, mean.p, 1);
  }
  // planes (kmeans.hpp:183-186)
  const uint64_t P = static_cast<uint64_t>(std::ceil(std::log2(4.0 * static_cast<double>(C))));
  if (P > 24) fail(kSize, "too many LSH planes (n_clusters too large)");
  std::vector<double> planes(P * d);
  for (double& w : planes) w = rng.gaussian();
  DBuf<double> planes_d(P * d);
  NB_CUDA(cudaMemcpyAsync(planes_d.p, planes.data(), P * d * 8, cudaMemcpyHostToDevice, S));
  // codes + buckets in code order, members ascending (the std::map)
  DBuf<uint32_t> codes(std::max<uint64_t>(n, 1));
  if (n) {
    k_lsh_hash<<<(unsigned)((n + 127) / 128), 128, 0, S>>>(km.x, n, (uint32_t)d, mean.p,
                                                           planes_d.p, (uint32_t)P, codes.p);
    note_launch(ctx, "k_lsh_hash");
  }
  const uint32_t L = 1u << P;
  DBuf<uint32_t> mem;
  std::vector<uint64_t> off;
  group_by_label(ctx, codes.p, n, L, mem, off);
  // bucket sizes over every rank (the std::map's, kmeans.hpp:189-201)
  std::vector<uint64_t> bsz(L);
  for (uint32_t c = 0; c < L; ++c) bsz[c] = off[c + 1] - off[c];
  if (km.comm) km.comm->allreduce_u64(bsz.data(), L);
  // rank: stable sort by size descending over ascending codes (kmeans.hpp:204-210)
  std::vector<uint32_t> ranked;
  for (uint32_t c = 0; c < L; ++c)
    if (bsz[c] > 0) ranked.push_back(c);
  std::stable_sort(ranked.begin(), ranked.end(),
                   [&](uint32_t a, uint32_t b) { return bsz[a] > bsz[b]; });
  const uint32_t seeded = std::min<uint32_t>(C, (uint32_t)ranked.size());
  NB_CUDA(cudaMemsetAsync(km.cent.p, 0, (uint64_t)C * d * 8, S));
  {
    std::vector<uint64_t> beg, cnt;
    std::vector<uint32_t> rows;
    std::vector<double> div(C, 0.0);
    for (uint32_t r = 0; r < seeded; ++r) {
      div[r] = (double)bsz[ranked[r]];
      if (off[ranked[r] + 1] > off[ranked[r]]) {
        beg.push_back(off[ranked[r]]);
        cnt.push_back(off[ranked[r] + 1] - off[ranked[r]]);
        rows.push_back(r);
      }
    }
    km.seq_means(mem.p, beg, cnt, rows, div, km.cent.p, C);  // kmeans.hpp:218-226
  }
  if (seeded < C) {  // kmeans.hpp:228-242 perturbation
    km.dist.alloc(std::max<uint64_t>(n, 1));
    if (n) {
      k_point_sqdist<<<(unsigned)((n + 127) / 128), 128, 0, S>>>(km.x, n, (uint32_t)d, mean.p,
                                                                nullptr, km.dist.p);
      note_launch(ctx, "k_point_sqdist");
    }
    double scale = km.seq_sum(km.dist.p);
    std::vector<double> c((uint64_t)C * d);
    NB_CUDA(cudaMemcpyAsync(c.data(), km.cent.p, c.size() * 8, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    scale = std::sqrt(scale / static_cast<double>(km.n_total)) * 1e-3 + 1e-12;
    uint64_t source = 0;
    for (uint64_t r = seeded; r < C; ++r) {
      for (uint64_t j = 0; j < d; ++j) c[r * d + j] = c[source * d + j] + scale * rng.gaussian();
      source = (source + 1) % seeded;
    }
    NB_CUDA(cudaMemcpyAsync(km.cent.p, c.data(), c.size() * 8, cudaMemcpyHostToDevice, S));
  }
  km.assign(false, nullptr);   // kmeans.hpp:244-246
  km.recompute_sizes();        // :247
  km.repair();                 // :248
}

// kmeans.hpp:257-296. tol_lo/tol_hi bracket the tolerance (equal when the
// caller passed an explicit tol); the exact value is only computed when a
// max_move falls inside the bracket.
uint64_t kmeans_em_dev(nomad_b200_ctx* ctx, KMeans& km, uint64_t max_iters, double tol_lo,
                       double tol_hi, bool auto_tol, double* qe_trace) {
  DBuf<double> prev((uint64_t)km.C * km.d), moves(km.C);
  std::vector<double> mv(km.C);
  double tol_exact = tol_lo;
  bool have_exact = !auto_tol;
  uint64_t it = 0;
  for (; it < max_iters; ++it) {
    unsigned long long changes = 0;
    km.assign(true, &changes);
    km.recompute_sizes();
    NB_CUDA(cudaMemcpyAsync(prev.p, km.cent.p, prev.bytes(), cudaMemcpyDeviceToDevice, km.S()));
    km.recompute_all();
    km.repair();
    k_moves<<<(km.C + 127) / 128, 128, 0, km.S()>>>(km.cent.p, prev.p, km.C, (uint32_t)km.d,
                                                    moves.p);
    note_launch(ctx, "k_moves");
    NB_CUDA(cudaMemcpyAsync(mv.data(), moves.p, km.C * 8, cudaMemcpyDeviceToHost, km.S()));
    NB_CUDA(cudaStreamSynchronize(km.S()));
    double max_move = 0.0;
    for (double m : mv) max_move = std::max(max_move, m);
    if (qe_trace) qe_trace[it] = km.quantization_error();
    bool below;
    if (have_exact) {
      below = max_move < tol_exact;
    } else if (max_move < tol_lo) {
      below = true;
    } else if (!(max_move < tol_hi)) {
      below = false;
    } else {
      tol_exact = default_tol_exact(ctx, km.x, km.n, km.d, km.comm, km.n_total);
      have_exact = true;
      below = max_move < tol_exact;
    }
    if (changes == 0 || below) {
      ++it;
      break;
    }
  }
  return it;
}

// Row-sharded lsh_init + kmeans_em (fit's call, optimizer.hpp:336-339; tol
// < 0: default_kmeans_tol) for this rank's rows [row0, row0 + n).
void sharded_kmeans(nomad_b200_ctx* ctx, Comm* comm, XPtr x, uint64_t n, uint64_t row0,
                    uint64_t n_total, uint64_t d, uint32_t C, uint64_t seed, uint64_t max_iters,
                    double tol, std::vector<uint32_t>& a_local, std::vector<double>& cent,
                    std::vector<uint32_t>& sizes) {
  if (C < 2 || C > n_total)
    fail(kParameter, "cluster count must be in [2, n]; got " + std::to_string(C));
  KMeans km(ctx, x, n, d, C);
  km.comm = comm;
  km.row0 = row0;
  km.n_total = n_total;
  lsh_init_dev(ctx, km, seed);
  if (tol >= 0.0) {
    kmeans_em_dev(ctx, km, max_iters, tol, tol, false, nullptr);
  } else {
    double lo = 0.0, hi = 0.0;
    default_tol_bracket(ctx, x, n, d, &lo, &hi, comm, n_total);
    kmeans_em_dev(ctx, km, max_iters, lo, hi, true, nullptr);
  }
  if (max_iters == 0) km.recompute_sizes();
  a_local.resize(n);
  cent.resize((size_t)C * d);
  NB_CUDA(cudaMemcpyAsync(a_local.data(), km.a.p, n * 4, cudaMemcpyDeviceToHost, km.S()));
  NB_CUDA(cudaMemcpyAsync(cent.data(), km.cent.p, cent.size() * 8, cudaMemcpyDeviceToHost, km.S()));
  NB_CUDA(cudaStreamSynchronize(km.S()));
  sizes = km.sizes;
}

}  // namespace nb

using namespace nb;

namespace {

void export_clusters(KMeans& km, nomad_b200_clusters* out) {
  cudaStream_t S = km.S();
  const auto kind = out->location == NOMAD_B200_DEVICE ? cudaMemcpyDeviceToDevice
                                                       : cudaMemcpyDeviceToHost;
  if (out->assignment)
    copy_out(km.ctx, out->assignment, km.a.p, km.n * 4, out->location == NOMAD_B200_DEVICE);
  if (out->centroids)
    NB_CUDA(cudaMemcpyAsync(out->centroids, km.cent.p, (uint64_t)km.C * km.d * 8, kind, S));
  if (out->sizes) NB_CUDA(cudaMemcpyAsync(out->sizes, km.sizes_d.p, km.C * 4, kind, S));
  NB_CUDA(cudaStreamSynchronize(S));
  out->rows = km.n;
  out->n_clusters = km.C;
  out->dims = km.d;
}

void import_clusters(KMeans& km, const nomad_b200_clusters* in) {
  cudaStream_t S = km.S();
  const auto kind = in->location == NOMAD_B200_DEVICE ? cudaMemcpyDeviceToDevice
                                                      : cudaMemcpyHostToDevice;
  if (!in->assignment || !in->centroids) fail(kParameter, "init assignment/centroids are NULL");
  if (in->location == NOMAD_B200_DEVICE)
    NB_CUDA(cudaMemcpyAsync(km.a.p, in->assignment, km.n * 4, kind, S));
  else
    copy_h2d(km.ctx, km.a.p, in->assignment, km.n * 4);
  NB_CUDA(cudaMemcpyAsync(km.cent.p, in->centroids, (uint64_t)km.C * km.d * 8, kind, S));
  NB_CUDA(cudaStreamSynchronize(S));
}

}  // namespace

extern "C" {

int32_t nomad_b200_default_kmeans_tol(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                      double* tol_out) {
  return guard([&] {
    if (!ctx || !tol_out) fail(kParameter, "NULL argument");
    bind_device(ctx);
    DevData dd;
    dd.bind(data, ctx);
    *tol_out = default_tol_exact(ctx, dd.x, dd.n, dd.d);
  });
}

int32_t nomad_b200_lsh_init(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                            uint64_t n_clusters, uint64_t seed, nomad_b200_clusters* out) {
  return guard([&] {
    if (!ctx || !out) fail(kParameter, "NULL argument");
    bind_device(ctx);
    DevData dd;
    dd.bind(data, ctx);
    if (n_clusters < 2 || n_clusters > dd.n)
      fail(kParameter, "cluster count must be in [2, n]; got " + std::to_string(n_clusters));
    KMeans km(ctx, dd.x, dd.n, dd.d, (uint32_t)n_clusters);
    lsh_init_dev(ctx, km, seed);
    export_clusters(km, out);
  });
}

int32_t nomad_b200_kmeans_em(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                             nomad_b200_clusters* inout, uint64_t max_iters, double tol,
                             double* qe_trace, uint64_t* iters_out) {
  return guard([&] {
    if (!ctx || !inout) fail(kParameter, "NULL argument");
    bind_device(ctx);
    DevData dd;
    dd.bind(data, ctx);
    if (inout->rows != dd.n || inout->dims != dd.d)
      fail(kParameter, "init assignment does not match dataset");
    if (inout->n_clusters < 1) fail(kParameter, "n_clusters must be >= 1");
    KMeans km(ctx, dd.x, dd.n, dd.d, (uint32_t)inout->n_clusters);
    import_clusters(km, inout);
    const uint64_t it = kmeans_em_dev(ctx, km, max_iters, tol, tol, false, qe_trace);
    if (max_iters == 0) km.recompute_sizes();
    export_clusters(km, inout);
    if (iters_out) *iters_out = it;
  });
}

int32_t nomad_b200_kmeans_em_default_tol(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                         nomad_b200_clusters* inout, uint64_t max_iters,
                                         double* qe_trace, uint64_t* iters_out) {
  return guard([&] {
    if (!ctx || !inout) fail(kParameter, "NULL argument");
    bind_device(ctx);
    DevData dd;
    dd.bind(data, ctx);
    if (inout->rows != dd.n || inout->dims != dd.d)
      fail(kParameter, "init assignment does not match dataset");
    if (inout->n_clusters < 1) fail(kParameter, "n_clusters must be >= 1");
    KMeans km(ctx, dd.x, dd.n, dd.d, (uint32_t)inout->n_clusters);
    import_clusters(km, inout);
    double lo = 0.0, hi = 0.0;
    default_tol_bracket(ctx, dd.x, dd.n, dd.d, &lo, &hi);
    const uint64_t it = kmeans_em_dev(ctx, km, max_iters, lo, hi, true, qe_trace);
    if (max_iters == 0) km.recompute_sizes();
    export_clusters(km, inout);
    if (iters_out) *iters_out = it;
  });
}

}  // extern "C"
