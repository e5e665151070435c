// Shared pieces of the index build (k-means partitioner, kNN graph):
// device-resident dataset views, the reference Rng on the host, stable
// grouping of points by label, exact sequential column sums.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <random>
#include <vector>

#include "common.cuh"
#include "hostcopy.cuh"

namespace nb {

__host__ __device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

// The reference's Rng (rng.hpp:25-84): splitmix stream seeds, mt19937_64,
// rejection-sampled bounded ints, 53-bit uniforms, Box-Muller with a cached
// spare. Host-side (it seeds the LSH planes and the perturbation draws,
// O(planes x d) values; libm gives the reference's bits on this image).
struct HostRng {
  std::mt19937_64 g;
  double spare = 0.0;
  bool have = false;
  static uint64_t mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
  }
  static uint64_t stream_seed(uint64_t base, uint64_t s) { return mix(base ^ mix(s)); }
  explicit HostRng(uint64_t seed) : g(seed) {}
  // unbiased integer in [0, n): rejection on the top range (rng.hpp:49-55)
  uint64_t uniform_index(uint64_t n) {
    const uint64_t limit = n * (0xFFFFFFFFFFFFFFFFull / n);
    uint64_t draw = g();
    while (draw >= limit) draw = g();
    return draw % n;
  }
  double uniform01() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
  double gaussian() {
    if (have) {
      have = false;
      return spare;
    }
    double u = uniform01();
    while (u == 0.0) u = uniform01();
    const double v = uniform01();
    const double radius = std::sqrt(-2.0 * std::log(u));
    const double angle = 6.283185307179586476925286766559 * v;
    spare = radius * std::sin(angle);
    have = true;
    return radius * std::cos(angle);
  }
};

// Reference fp64 distance (knn.hpp:51-58), j ascending, no FMA.
__device__ __forceinline__ double ref_dist(const float* __restrict__ a, const float* __restrict__ b,
                                           uint32_t d) {
  double acc = 0.0;
  uint32_t j = 0;
  if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0) {
    for (; j + 4 <= d; j += 4) {
      const float4 u = *reinterpret_cast<const float4*>(a + j);
      const float4 v = *reinterpret_cast<const float4*>(b + j);
      double t = __dsub_rn((double)u.x, (double)v.x);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
      t = __dsub_rn((double)u.y, (double)v.y);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
      t = __dsub_rn((double)u.z, (double)v.z);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
      t = __dsub_rn((double)u.w, (double)v.w);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
  }
  for (; j < d; ++j) {
    const double t = __dsub_rn((double)a[j], (double)b[j]);
    acc = __dadd_rn(acc, __dmul_rn(t, t));
  }
  return acc;
}

__device__ __forceinline__ bool key_less(double da, uint32_t ia, double db, uint32_t ib) {
  return da < db || (da == db && ia < ib);
}

// A dataset on the device (uploaded once per call when the caller passed
// host memory).
// Dataset rows as kernels read them: f32 (the reference's VectorDataset) or
// bf16 (large configurations); elements widen exactly to float, so every
// kernel computes the same values as on the widened f32 data.
struct XPtr {
  const void* p = nullptr;
  int bf = 0;
  XPtr() = default;
  __host__ __device__ XPtr(const float* f) : p(f), bf(0) {}  // NOLINT: f32 rows
  __host__ __device__ XPtr(const void* q, int b) : p(q), bf(b) {}
  __host__ __device__ XPtr operator+(uint64_t o) const {
    XPtr r = *this;
    r.p = bf ? (const void*)(static_cast<const __nv_bfloat16*>(p) + o)
             : (const void*)(static_cast<const float*>(p) + o);
    return r;
  }
  __device__ __forceinline__ float operator[](uint64_t i) const {
    return bf ? __bfloat162float(__ldg(static_cast<const __nv_bfloat16*>(p) + i))
              : __ldg(static_cast<const float*>(p) + i);
  }
};

// ref_dist on dataset rows (both rows of one dataset)
__device__ __forceinline__ double ref_dist(XPtr a, XPtr b, uint32_t d) {
  if (!a.bf) return ref_dist(static_cast<const float*>(a.p), static_cast<const float*>(b.p), d);
  double acc = 0.0;
  for (uint32_t j = 0; j < d; ++j) {
    const double t = __dsub_rn((double)a[j], (double)b[j]);
    acc = __dadd_rn(acc, __dmul_rn(t, t));
  }
  return acc;
}

// f32 rows for the kernels that stage f32 directly (loud failure for bf16)
inline const float* need_f32(XPtr x, const char* what) {
  if (x.bf) fail(kParameter, std::string(what) + ": bf16 datasets are not supported here");
  return static_cast<const float*>(x.p);
}

struct DevData {
  XPtr x;
  uint64_t n = 0, d = 0;
  DBuf<float> owned;
  DBuf<uint16_t> owned16;
  // host rows are uploaded through the context's pinned staging ring
  void bind(const nomad_b200_dataset_view* v, nomad_b200_ctx* ctx) {
    if (!v || !v->data) fail(kParameter, "dataset view is NULL");
    n = v->rows;
    d = v->dims;
    if (n < 1 || d < 1) fail(kParameter, "empty dataset");
    if (n >= 0xFFFFFFFFull) fail(kSize, "point ids are u32 (n < 2^32)");
    if (v->dtype != NOMAD_B200_F32 && v->dtype != NOMAD_B200_BF16)
      fail(kParameter, "dataset dtype must be NOMAD_B200_F32 or NOMAD_B200_BF16");
    x.bf = v->dtype == NOMAD_B200_BF16;
    if (v->location == NOMAD_B200_DEVICE) {
      x.p = v->data;
    } else if (x.bf) {
      owned16.alloc(n * d);
      copy_h2d(ctx, owned16.p, v->data, n * d * 2);
      x.p = owned16.p;
    } else {
      owned.alloc(n * d);
      copy_h2d(ctx, owned.p, v->data, n * d * 4);
      x.p = owned.p;
    }
  }
  // f32 rows for the paths that take only f32 (loud failure for bf16)
  const float* f32(const char* what) const {
    if (x.bf) fail(kParameter, std::string(what) + ": bf16 datasets are not supported here");
    return static_cast<const float*>(x.p);
  }
};

// Stable grouping of [0, n) by label (labels >= L are dropped): members of
// label r are written to members[off[r] .. off[r+1]) in ascending id order.
// off (host) receives L + 1 offsets.
void group_by_label(nomad_b200_ctx* ctx, const uint32_t* labels, uint64_t n, uint32_t L,
                    DBuf<uint32_t>& members, std::vector<uint64_t>& off);

// out[seg_ids[s] * d + j] = (sum over members[beg[s] .. beg[s] + cnt[s]),
// in order, of (double) x[m * d + j]) / cnt[s]  — the reference's sequential centroid /
// mean accumulation (kmeans.hpp:75-104, :176-181, :218-226) bit for bit.
// members == nullptr means the identity list. Segments with count 0 are
// left untouched. carry: `out` holds running sums that the segments continue
// (a row-sharded build's carry chain, shard.cuh), written back undivided.
void seq_column_means(nomad_b200_ctx* ctx, XPtr x, uint64_t d, const uint32_t* members,
                      const std::vector<uint64_t>& beg, const std::vector<uint64_t>& cnt,
                      const std::vector<uint32_t>& seg_ids, double* out, bool carry = false);
// Same outputs up to rounding, summed in a fixed parallel order (1024-row
// chunks): for centres that only need to be fixed, not the reference's value.
void fast_column_means(nomad_b200_ctx* ctx, XPtr x, uint64_t d, const uint32_t* members,
                       const std::vector<uint64_t>& beg, const std::vector<uint64_t>& cnt,
                       const std::vector<uint32_t>& seg_ids, double* out);

// Exact global kNN of m sampled points (knn.cu): out_ids_d[v * k + r] = the
// r-th smallest (reference fp64 distance, id) key of point qlist_d[v] among
// all other points. 1 <= k <= 56, k < n.
void knn_global_sample(nomad_b200_ctx* ctx, XPtr x, uint64_t n, uint64_t d,
                       const uint32_t* qlist_d, uint32_t m, uint32_t k, uint32_t* out_ids_d);

}  // namespace nb
