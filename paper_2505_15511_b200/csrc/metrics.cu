// Final-map quality metrics on the GPU (metrics.hpp:113-243):
// neighbourhood preservation NP@k (exact, and NP-ann against a prebuilt
// graph) and random-triplet accuracy.
//
// Both keep the reference's sampling streams (drawn on the host with the
// reference Rng: stream_seed(seed, "np") partial Fisher-Yates, :127-136;
// stream_seed(seed, "tri") rejection triplets, :215-222), its distance chains
// (sq_dist_rows: fp64 j-ascending, no FMA, :57-64; sq_dist_2d, :66-70) and
// its tie rule (partial_sort on (distance, id), :77-91), and accumulate in
// evaluation order, so value and std_error are bit-identical to the
// reference's. The O(sample x n x d) search runs on the device:
//  * high-d: knn_global_sample (knn.cu) — FFMA certified filter over all
//    points, fp64 re-rank, exhaustive fp64 for the rows it cannot certify;
//  * 2-D: k_np_low_partial — each thread scans a candidate partition for one
//    sampled point in fp64, keeping a sorted top-k; k_np_low_merge merges
//    the partitions;
//  * triplets: k_triplet, one thread per triplet, integer agreement count.
#include <algorithm>
#include <cmath>
#include <numeric>

#include "index_common.cuh"

namespace nb {

namespace {

constexpr int LKMAX = 1024;  // k bound (k <= 56: the certified filter + register lists;
                             // larger k: exhaustive high-d rows, local-memory lists)
constexpr int LTILE = 1024; // layout rows per shared-memory tile

__device__ __forceinline__ double sq_dist_2d(double ax, double ay, double bx, double by) {
  const double dx = __dsub_rn(ax, bx), dy = __dsub_rn(ay, by);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// grid (ceil(m / 128), P): thread = sampled slot v, blockIdx.y = candidate
// partition [n p / P, n (p + 1) / P). Output: the partition's k smallest
// (distance, id) keys of slot v, sorted, padded with (+inf, ~0).
template <int LK>
__global__ void __launch_bounds__(128) k_np_low_partial(const double* __restrict__ lay, uint64_t n,
                                                        const uint32_t* __restrict__ qlist,
                                                        uint32_t m, uint32_t k, uint32_t P,
                                                        double* pd, uint32_t* pi) {
  __shared__ double tx[LTILE], ty[LTILE];
  const uint32_t v = blockIdx.x * 128 + threadIdx.x;
  const uint32_t p = blockIdx.y;
  const uint64_t lo = n * p / P, hi = n * (p + 1) / P;
  const bool valid = v < m;
  const uint32_t q = valid ? qlist[v] : 0u;
  const double qx = valid ? lay[2 * (uint64_t)q] : 0.0, qy = valid ? lay[2 * (uint64_t)q + 1] : 0.0;
  double bd[LK];
  uint32_t bi[LK];
  uint32_t cnt = 0;
  for (uint64_t t0 = lo; t0 < hi; t0 += LTILE) {
    __syncthreads();
    for (int e = threadIdx.x; e < LTILE; e += 128) {
      const uint64_t j = t0 + e;
      tx[e] = j < hi ? lay[2 * j] : 0.0;
      ty[e] = j < hi ? lay[2 * j + 1] : 0.0;
    }
    __syncthreads();
    if (!valid) continue;
    const int lim = (int)umin64(LTILE, hi - t0);
    for (int e = 0; e < lim; ++e) {
      const uint32_t j = (uint32_t)(t0 + e);
      const double dd = sq_dist_2d(qx, qy, tx[e], ty[e]);
      if (cnt == k && !key_less(dd, j, bd[k - 1], bi[k - 1])) continue;
      if (j == q) continue;
      uint32_t pos = cnt < k ? cnt : k - 1;
      while (pos > 0 && key_less(dd, j, bd[pos - 1], bi[pos - 1])) {
        bd[pos] = bd[pos - 1];
        bi[pos] = bi[pos - 1];
        --pos;
      }
      bd[pos] = dd;
      bi[pos] = j;
      if (cnt < k) ++cnt;
    }
  }
  if (!valid) return;
  const uint64_t o = ((uint64_t)v * P + p) * k;
  for (uint32_t r = 0; r < k; ++r) {
    pd[o + r] = r < cnt ? bd[r] : __longlong_as_double(0x7ff0000000000000ll);
    pi[o + r] = r < cnt ? bi[r] : 0xFFFFFFFFu;
  }
}

void np_low_partial(dim3 grid, cudaStream_t S, const double* lay, uint64_t n, const uint32_t* ql,
                    uint32_t m, uint32_t k, uint32_t P, double* pd, uint32_t* pi) {
  if (k <= 56)
    k_np_low_partial<56><<<grid, 128, 0, S>>>(lay, n, ql, m, k, P, pd, pi);
  else if (k <= 256)
    k_np_low_partial<256><<<grid, 128, 0, S>>>(lay, n, ql, m, k, P, pd, pi);
  else
    k_np_low_partial<1024><<<grid, 128, 0, S>>>(lay, n, ql, m, k, P, pd, pi);
}

// thread per slot: P-way merge of the sorted partition lists, first k keys.
__global__ void k_np_low_merge(uint32_t m, uint32_t k, uint32_t P, const double* pd,
                               const uint32_t* pi, uint32_t* out) {
  const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= m) return;
  uint32_t head[64];
  for (uint32_t p = 0; p < P; ++p) head[p] = 0;
  const uint64_t base = (uint64_t)v * P * k;
  for (uint32_t r = 0; r < k; ++r) {
    uint32_t bp = 0;
    double bdv = __longlong_as_double(0x7ff0000000000000ll);
    uint32_t bid = 0xFFFFFFFFu;
    for (uint32_t p = 0; p < P; ++p) {
      if (head[p] >= k) continue;
      const uint64_t e = base + (uint64_t)p * k + head[p];
      if (key_less(pd[e], pi[e], bdv, bid)) {
        bdv = pd[e];
        bid = pi[e];
        bp = p;
      }
    }
    ++head[bp];
    out[(uint64_t)v * k + r] = bid;
  }
}

// thread per triplet (a, b, c): agreement of the two orderings (:229-235).
__global__ void k_triplet(XPtr x, uint32_t d, const double* __restrict__ lay,
                          const uint32_t* __restrict__ trip, uint64_t T,
                          unsigned long long* agree) {
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t ok = 0;
  if (t < T) {
    const uint64_t a = trip[3 * t], b = trip[3 * t + 1], c = trip[3 * t + 2];
    const double hab = ref_dist(x + a * d, x + b * d, d);
    const double hac = ref_dist(x + a * d, x + c * d, d);
    const double lab = sq_dist_2d(lay[2 * a], lay[2 * a + 1], lay[2 * b], lay[2 * b + 1]);
    const double lac = sq_dist_2d(lay[2 * a], lay[2 * a + 1], lay[2 * c], lay[2 * c + 1]);
    const int ho = hab < hac ? -1 : (hab > hac ? 1 : 0);
    const int lo = lab < lac ? -1 : (lab > lac ? 1 : 0);
    ok = ho == lo ? 1u : 0u;
  }
  for (int o = 16; o > 0; o >>= 1) ok += __shfl_xor_sync(0xffffffffu, ok, o);
  if ((threadIdx.x & 31) == 0 && ok) atomicAdd(agree, (unsigned long long)ok);
}

// A layout on the device (uploaded when the caller passed host memory).
struct DevLayout {
  const double* p = nullptr;
  DBuf<double> owned;
  void bind(const double* lay, int32_t loc, uint64_t n, cudaStream_t S) {
    if (!lay) fail(kParameter, "layout is NULL");
    if (loc == NOMAD_B200_DEVICE) {
      p = lay;
    } else {
      owned.alloc(2 * n);
      NB_CUDA(cudaMemcpyAsync(owned.p, lay, 2 * n * 8, cudaMemcpyHostToDevice, S));
      p = owned.p;
    }
  }
};

}  // namespace

}  // namespace nb

using namespace nb;

extern "C" {

int32_t nomad_b200_neighborhood_preservation(nomad_b200_ctx* ctx,
                                             const nomad_b200_dataset_view* high,
                                             const double* layout, int32_t layout_location,
                                             uint64_t k, uint64_t sample, uint64_t seed,
                                             double* value, double* std_error) {
  return guard([&] {
    if (!ctx || !value) fail(kParameter, "NULL argument");
    bind_device(ctx);
    cudaStream_t S = ctx->stream;
    DevData dd;
    dd.bind(high, ctx);
    const uint64_t n = dd.n;
    if (k >= n) fail(kParameter, "k must be < n");
    if (k < 1 || k > (uint64_t)LKMAX)
      fail(kParameter, "GPU neighborhood_preservation supports 1 <= k <= 1024");
    DevLayout L;
    L.bind(layout, layout_location, n, S);
    // evaluated points (metrics.hpp:122-136)
    std::vector<uint32_t> ev;
    if (sample == 0 || sample >= n) {
      ev.resize(n);
      std::iota(ev.begin(), ev.end(), 0u);
      sample = 0;
    } else {
      std::vector<uint32_t> pool(n);
      std::iota(pool.begin(), pool.end(), 0u);
      HostRng rng(HostRng::stream_seed(seed, 0x6e70));
      for (uint64_t t = 0; t < sample; ++t) {
        const uint64_t pick = t + rng.uniform_index(n - t);
        std::swap(pool[t], pool[pick]);
        ev.push_back(pool[t]);
      }
    }
    const uint32_t m = (uint32_t)ev.size();
    DBuf<uint32_t> ql(m), hi_ids((uint64_t)m * k), lo_ids((uint64_t)m * k);
    NB_CUDA(cudaMemcpyAsync(ql.p, ev.data(), (uint64_t)m * 4, cudaMemcpyHostToDevice, S));
    knn_global_sample(ctx, dd.x, n, dd.d, ql.p, m, (uint32_t)k, hi_ids.p);
    {
      const uint32_t bx = (m + 127) / 128;
      uint32_t P = 1;
      while (P < 64 && bx * P < 4 * (uint32_t)ctx->sm_count && n / (2 * P) >= 4096) P *= 2;
      DBuf<double> pd((uint64_t)m * P * k);
      DBuf<uint32_t> pi((uint64_t)m * P * k);
      np_low_partial(dim3(bx, P), S, L.p, n, ql.p, m, (uint32_t)k, P, pd.p, pi.p);
      note_launch(ctx, "k_np_low_partial");
      k_np_low_merge<<<(m + 127) / 128, 128, 0, S>>>(m, (uint32_t)k, P, pd.p, pi.p, lo_ids.p);
      note_launch(ctx, "k_np_low_merge");
      std::vector<uint32_t> hh((uint64_t)m * k), lh((uint64_t)m * k);
      NB_CUDA(cudaMemcpyAsync(hh.data(), hi_ids.p, hh.size() * 4, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaMemcpyAsync(lh.data(), lo_ids.p, lh.size() * 4, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
      // overlap per evaluated point, accumulated in evaluation order (:138-150)
      double sum = 0.0, sum_sq = 0.0;
      for (uint64_t v = 0; v < m; ++v) {
        uint32_t* a = hh.data() + v * k;
        uint32_t* b = lh.data() + v * k;
        std::sort(a, a + k);
        std::sort(b, b + k);
        uint64_t count = 0, ia = 0, ib = 0;
        while (ia < k && ib < k) {
          if (a[ia] < b[ib]) ++ia;
          else if (b[ib] < a[ia]) ++ib;
          else ++count, ++ia, ++ib;
        }
        const double overlap = static_cast<double>(count) / static_cast<double>(k);
        sum += overlap;
        sum_sq += overlap * overlap;
      }
      const double cntd = static_cast<double>(m);
      *value = sum / cntd;
      double se = 0.0;
      if (sample != 0 && m > 1) {
        const double var = std::max(0.0, sum_sq / cntd - *value * *value);
        se = std::sqrt(var / cntd);
      }
      if (std_error) *std_error = se;
    }
  });
}

int32_t nomad_b200_neighborhood_preservation_ann(nomad_b200_ctx* ctx,
                                                 const nomad_b200_graph* graph,
                                                 const double* layout, int32_t layout_location,
                                                 uint64_t k, double* value) {
  return guard([&] {
    if (!ctx || !graph || !value || !graph->offsets) fail(kParameter, "NULL argument");
    bind_device(ctx);
    cudaStream_t S = ctx->stream;
    const uint64_t n = graph->rows;
    if (k >= n) fail(kParameter, "k must be < n");
    if (k < 1 || k > (uint64_t)LKMAX)
      fail(kParameter, "GPU neighborhood_preservation_ann supports 1 <= k <= 1024");
    if (n >= 0xFFFFFFFFull) fail(kSize, "point ids are u32 (n < 2^32)");
    DevLayout L;
    L.bind(layout, layout_location, n, S);
    // graph lists on the host (the intersection runs there, in row order)
    std::vector<uint32_t> off(n + 1), nbh;
    const bool dev = graph->location == NOMAD_B200_DEVICE;
    NB_CUDA(cudaMemcpy(off.data(), graph->offsets, (n + 1) * 4,
                       dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
    nbh.resize(std::max<uint64_t>(off[n], 1));
    if (off[n])
      NB_CUDA(cudaMemcpy(nbh.data(), graph->neighbors, (uint64_t)off[n] * 4,
                         dev ? cudaMemcpyDeviceToHost : cudaMemcpyHostToHost));
    // exact 2-D neighbours of every row (metrics.hpp:187-189), in row batches
    const uint64_t B = 1ull << 22;
    DBuf<uint32_t> ql(std::min(B, n)), lo_ids(std::min(B, n) * k);
    std::vector<uint32_t> lh, idx(std::min(B, n));
    double sum = 0.0;
    for (uint64_t r0 = 0; r0 < n; r0 += B) {
      const uint32_t m = (uint32_t)std::min(B, n - r0);
      for (uint32_t v = 0; v < m; ++v) idx[v] = (uint32_t)(r0 + v);
      NB_CUDA(cudaMemcpyAsync(ql.p, idx.data(), (uint64_t)m * 4, cudaMemcpyHostToDevice, S));
      const uint32_t bx = (m + 127) / 128;
      uint32_t P = 1;
      while (P < 64 && bx * P < 4 * (uint32_t)ctx->sm_count && n / (2 * P) >= 4096) P *= 2;
      DBuf<double> pd((uint64_t)m * P * k);
      DBuf<uint32_t> pi((uint64_t)m * P * k);
      np_low_partial(dim3(bx, P), S, L.p, n, ql.p, m, (uint32_t)k, P, pd.p, pi.p);
      note_launch(ctx, "k_np_low_partial");
      k_np_low_merge<<<(m + 127) / 128, 128, 0, S>>>(m, (uint32_t)k, P, pd.p, pi.p, lo_ids.p);
      note_launch(ctx, "k_np_low_merge");
      lh.resize((uint64_t)m * k);
      NB_CUDA(cudaMemcpyAsync(lh.data(), lo_ids.p, lh.size() * 4, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
      std::vector<uint32_t> hi;
      for (uint32_t v = 0; v < m; ++v) {  // metrics.hpp:182-191, row order
        const uint64_t i = r0 + v;
        const uint64_t have = std::min<uint64_t>(k, off[i + 1] - off[i]);
        hi.assign(nbh.begin() + off[i], nbh.begin() + off[i] + have);
        std::sort(hi.begin(), hi.end());
        uint32_t* b = lh.data() + (uint64_t)v * k;
        std::sort(b, b + k);
        uint64_t count = 0, ia = 0, ib = 0;
        while (ia < hi.size() && ib < k) {
          if (hi[ia] < b[ib]) ++ia;
          else if (b[ib] < hi[ia]) ++ib;
          else ++count, ++ia, ++ib;
        }
        sum += static_cast<double>(count) / static_cast<double>(k);
      }
    }
    *value = sum / static_cast<double>(n);
  });
}

int32_t nomad_b200_random_triplet_accuracy(nomad_b200_ctx* ctx,
                                           const nomad_b200_dataset_view* high,
                                           const double* layout, int32_t layout_location,
                                           uint64_t n_triplets, uint64_t seed, double* value,
                                           double* std_error) {
  return guard([&] {
    if (!ctx || !value) fail(kParameter, "NULL argument");
    bind_device(ctx);
    cudaStream_t S = ctx->stream;
    DevData dd;
    dd.bind(high, ctx);
    const uint64_t n = dd.n;
    if (n < 3) fail(kParameter, "need at least 3 points");
    if (n_triplets < 1) fail(kParameter, "need at least 1 triplet");
    DevLayout L;
    L.bind(layout, layout_location, n, S);
    HostRng rng(HostRng::stream_seed(seed, 0x747269));
    DBuf<unsigned long long> agree(1);
    NB_CUDA(cudaMemsetAsync(agree.p, 0, 8, S));
    const uint64_t CH = 1ull << 22;  // triplets per device batch
    std::vector<uint32_t> th;
    DBuf<uint32_t> td(3 * std::min(CH, n_triplets));
    for (uint64_t t0 = 0; t0 < n_triplets; t0 += CH) {
      const uint64_t T = std::min(CH, n_triplets - t0);
      NB_CUDA(cudaStreamSynchronize(S));  // td is reused
      th.resize(3 * T);
      for (uint64_t t = 0; t < T; ++t) {  // :216-222
        const uint64_t a = rng.uniform_index(n);
        uint64_t b = rng.uniform_index(n);
        while (b == a) b = rng.uniform_index(n);
        uint64_t c = rng.uniform_index(n);
        while (c == a || c == b) c = rng.uniform_index(n);
        th[3 * t] = (uint32_t)a;
        th[3 * t + 1] = (uint32_t)b;
        th[3 * t + 2] = (uint32_t)c;
      }
      NB_CUDA(cudaMemcpyAsync(td.p, th.data(), 3 * T * 4, cudaMemcpyHostToDevice, S));
      k_triplet<<<(unsigned)((T + 255) / 256), 256, 0, S>>>(dd.x, (uint32_t)dd.d, L.p, td.p, T,
                                                            agree.p);
      note_launch(ctx, "k_triplet");
    }
    unsigned long long ag = 0;
    NB_CUDA(cudaMemcpyAsync(&ag, agree.p, 8, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    *value = static_cast<double>(ag) / static_cast<double>(n_triplets);
    if (std_error)
      *std_error = std::sqrt(*value * (1.0 - *value) / static_cast<double>(n_triplets));
  });
}

}  // extern "C"
