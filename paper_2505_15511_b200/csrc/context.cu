// Context, error plumbing, config defaults, NCCL id, device data generator.
#include <cuda_bf16.h>
#include <nccl.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "hostcopy.cuh"
#include "philox.cuh"

namespace nb {

static thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

void bind_device(nomad_b200_ctx* c) { NB_CUDA(cudaSetDevice(c->device)); }

namespace {
// Device allocations are cached: on this driver every cudaMalloc / cudaFree
// costs ~2 ms even for a 1 MB block (NOMAD_B200_DEBUG_ALLOC, profiles/
// r2_knn_wall.txt), and the index build makes hundreds of them. Blocks
// >= 64 MB are reused for requests in [size / 1.5, size]; smaller ones are
// rounded up to power-of-two classes and reused within their class.
constexpr size_t kCacheMin = 64ull << 20;   // large blocks: best fit
constexpr size_t kCacheCap = 24ull << 30;   // cached large bytes per device
constexpr size_t kSmallCap = 2ull << 30;    // cached small bytes per device
struct Cached {
  void* p;
  size_t bytes;
};
std::mutex g_cache_mu;
std::vector<Cached> g_cache[64];  // per device, large blocks
size_t g_cached[64];
std::vector<void*> g_small[64][32];  // per device, per power-of-two class (2^9 .. 2^26 bytes)
size_t g_small_bytes[64];

size_t small_class(size_t bytes, int* ci) {
  int c = 9;
  while (((size_t)1 << c) < bytes) ++c;
  *ci = c;
  return (size_t)1 << c;
}

// NOMAD_B200_DEBUG_ALLOC: report driver allocations / frees slower than 2 ms
bool alloc_dbg() {
  static const bool on = std::getenv("NOMAD_B200_DEBUG_ALLOC") != nullptr;
  return on;
}
struct SlowCall {
  const char* what;
  size_t bytes;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  ~SlowCall() {
    if (!alloc_dbg()) return;
    const double ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms > 2.0) std::fprintf(stderr, "alloc: %s %zu MB took %.1f ms\n", what, bytes >> 20, ms);
  }
};

void flush_cache(int dev) {  // caller holds the lock
  for (auto& c : g_cache[dev]) cudaFree(c.p);
  g_cache[dev].clear();
  g_cached[dev] = 0;
  for (auto& cl : g_small[dev]) {
    for (void* q : cl) cudaFree(q);
    cl.clear();
  }
  g_small_bytes[dev] = 0;
}
}  // namespace

void* dev_alloc(size_t bytes) {
  int dev = 0;
  NB_CUDA(cudaGetDevice(&dev));
  size_t want = bytes;
  if (dev < 64) {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    if (bytes >= kCacheMin) {
      auto& v = g_cache[dev];
      size_t best = v.size();
      for (size_t i = 0; i < v.size(); ++i)  // smallest block in [bytes, 1.5 bytes]
        if (v[i].bytes >= bytes && v[i].bytes <= bytes + bytes / 2 &&
            (best == v.size() || v[i].bytes < v[best].bytes))
          best = i;
      if (best != v.size()) {
        void* p = v[best].p;
        g_cached[dev] -= v[best].bytes;
        v.erase(v.begin() + best);
        return p;
      }
    } else {
      int ci = 0;
      want = small_class(bytes, &ci);
      auto& cl = g_small[dev][ci];
      if (!cl.empty()) {
        void* p = cl.back();
        cl.pop_back();
        g_small_bytes[dev] -= want;
        return p;
      }
    }
  }
  void* p = nullptr;
  SlowCall sc{"cudaMalloc", want};
  cudaError_t e = cudaMalloc(&p, want);
  if (e == cudaErrorMemoryAllocation && dev < 64) {
    cudaGetLastError();
    {
      std::lock_guard<std::mutex> lk(g_cache_mu);
      flush_cache(dev);
    }
    e = cudaMalloc(&p, want);
  }
  if (e != cudaSuccess)
    fail(kInternal, std::string("CUDA error ") + cudaGetErrorString(e) + " allocating " +
                        std::to_string(bytes) + " bytes");
  return p;
}

void dev_free(void* p, size_t bytes) {
  int dev = 0;
  SlowCall sc{"free", bytes};
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64 || bytes > kCacheCap) {
    cudaFree(p);
    return;
  }
  // a block is reused only once every kernel that may still touch it is done
  // (cudaFree would synchronise the device as well)
  if (cudaDeviceSynchronize() != cudaSuccess) {
    cudaFree(p);
    return;
  }
  std::lock_guard<std::mutex> lk(g_cache_mu);
  if (bytes < kCacheMin) {
    int ci = 0;
    const size_t cls = small_class(bytes, &ci);
    if (g_small_bytes[dev] + cls > kSmallCap) {
      cudaFree(p);
      return;
    }
    g_small[dev][ci].push_back(p);
    g_small_bytes[dev] += cls;
    return;
  }
  auto& v = g_cache[dev];
  while (!v.empty() && g_cached[dev] + bytes > kCacheCap) {  // evict the oldest
    cudaFree(v.front().p);
    g_cached[dev] -= v.front().bytes;
    v.erase(v.begin());
  }
  v.push_back(Cached{p, bytes});
  g_cached[dev] += bytes;
}

void note_launch(nomad_b200_ctx* c, const char* name) {
  ++c->launches;
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess)
    fail(kInternal, std::string("launch of ") + name + " failed: " + cudaGetErrorString(e));
}

// SURVEY §8(d) synthetic mixture: centres ~ N(0, spread^2 I), x_i =
// c_{i mod blobs} + N(0, I). Each thread emits 4 consecutive coordinates of
// one row from one Philox block (Box-Muller on two pairs, fp32).
__global__ void k_mixture_centres(float* centres, uint64_t count, float spread,
                                  uint32_t s0, uint32_t s1) {
  const uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (q * 4 >= count) return;
  const u32x4 r = philox4x32_10(u32x4{(uint32_t)q, (uint32_t)(q >> 32), 0xC3u, 0u}, s0, s1);
  const float u0 = ((r.x >> 8) + 1) * 0x1p-24f, v0 = (r.y >> 8) * 0x1p-24f;
  const float u1 = ((r.z >> 8) + 1) * 0x1p-24f, v1 = (r.w >> 8) * 0x1p-24f;
  const float a = sqrtf(-2.f * logf(u0)), b = sqrtf(-2.f * logf(u1));
  float g[4];
  sincospif(2.f * v0, &g[1], &g[0]);
  sincospif(2.f * v1, &g[3], &g[2]);
  g[0] *= a; g[1] *= a; g[2] *= b; g[3] *= b;
  for (int t = 0; t < 4; ++t)
    if (q * 4 + t < count) centres[q * 4 + t] = spread * g[t];
}

template <class T>
__device__ __forceinline__ T to_out(float v);
template <>
__device__ __forceinline__ float to_out<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 to_out<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// T = __nv_bfloat16: the same f32 values rounded to nearest-even bf16.
// Rows [row0, row0 + rows) of the mixture: element e of the full matrix is
// value e % 4 of Philox block e / 4, so any row slice (one rank's share of a
// row-sharded dataset) holds exactly the full matrix's values.
template <class T>
__global__ void k_mixture_points(T* out, const float* centres, uint64_t row0, uint64_t rows,
                                 uint64_t dims, uint64_t blobs, uint32_t s0, uint32_t s1) {
  const uint64_t base = row0 * dims, total = rows * dims;
  if (base & 3) {  // slice not aligned to a Philox block: per element
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
         e += (uint64_t)gridDim.x * blockDim.x) {
      const uint64_t ge = base + e, q = ge / 4;
      const u32x4 r = philox4x32_10(u32x4{(uint32_t)q, (uint32_t)(q >> 32), 0x9Au, 1u}, s0, s1);
      const float u0 = ((r.x >> 8) + 1) * 0x1p-24f, v0 = (r.y >> 8) * 0x1p-24f;
      const float u1 = ((r.z >> 8) + 1) * 0x1p-24f, v1 = (r.w >> 8) * 0x1p-24f;
      const float a = sqrtf(-2.f * __logf(u0)), b = sqrtf(-2.f * __logf(u1));
      float g[4];
      sincospif(2.f * v0, &g[1], &g[0]);
      sincospif(2.f * v1, &g[3], &g[2]);
      g[0] *= a; g[1] *= a; g[2] *= b; g[3] *= b;
      const uint64_t i = ge / dims, j = ge % dims;
      out[e] = to_out<T>(centres[(i % blobs) * dims + j] + g[ge & 3]);
    }
    return;
  }
  out -= base;  // index by global element below (only [base, base + total) is written)
  for (uint64_t q = base / 4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
       q * 4 < base + total; q += (uint64_t)gridDim.x * blockDim.x) {
    const u32x4 r = philox4x32_10(u32x4{(uint32_t)q, (uint32_t)(q >> 32), 0x9Au, 1u}, s0, s1);
    const float u0 = ((r.x >> 8) + 1) * 0x1p-24f, v0 = (r.y >> 8) * 0x1p-24f;
    const float u1 = ((r.z >> 8) + 1) * 0x1p-24f, v1 = (r.w >> 8) * 0x1p-24f;
    const float a = sqrtf(-2.f * __logf(u0)), b = sqrtf(-2.f * __logf(u1));
    float g[4];
    sincospif(2.f * v0, &g[1], &g[0]);
    sincospif(2.f * v1, &g[3], &g[2]);
    g[0] *= a; g[1] *= a; g[2] *= b; g[3] *= b;
    const uint64_t e0 = q * 4;
    if ((dims & 3) == 0 && e0 + 3 < base + total) {
      const uint64_t i = e0 / dims, j = e0 % dims;
      const float4 c = *reinterpret_cast<const float4*>(centres + (i % blobs) * dims + j);
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(out + e0) =
            make_float4(c.x + g[0], c.y + g[1], c.z + g[2], c.w + g[3]);
      } else {
        out[e0] = to_out<T>(c.x + g[0]);
        out[e0 + 1] = to_out<T>(c.y + g[1]);
        out[e0 + 2] = to_out<T>(c.z + g[2]);
        out[e0 + 3] = to_out<T>(c.w + g[3]);
      }
    } else {
      for (int t = 0; t < 4; ++t) {
        const uint64_t e = e0 + t;
        if (e >= base + total) break;
        const uint64_t i = e / dims, j = e % dims;
        out[e] = to_out<T>(centres[(i % blobs) * dims + j] + g[t]);
      }
    }
  }
}

}  // namespace nb

using namespace nb;

extern "C" {

const char* nomad_b200_last_error(void) { return g_last_error.c_str(); }

void nomad_b200_default_config(nomad_b200_train_config* c) {
  std::memset(c, 0, sizeof *c);
  c->epochs = 200;
  c->k = 15;
  c->negatives = 5;
  c->local_draws = 5;
  c->batch_size = 1024;
  c->workers = 1;
  c->n_clusters = 0;
  c->seed = 0;
  c->lr0 = 0.0;
  c->kmeans_max_iters = 100;
  c->kmeans_tol = -1.0;
  c->sgd_mode = NOMAD_B200_SGD_REPLAY;
  c->knn_mode = NOMAD_B200_KNN_EXACT;
  c->hogwild_cap = 0;
}

int32_t nomad_b200_create(int32_t device, nomad_b200_ctx** out) {
  return guard([&] {
    if (!out) fail(kParameter, "out is NULL");
    int n = 0;
    NB_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n)
      fail(kParameter, "device " + std::to_string(device) + " out of range (" +
                           std::to_string(n) + " visible)");
    cudaDeviceProp prop;
    NB_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
      fail(kConfig, std::string("libnomad_b200 is built for sm_100a; device is ") +
                        prop.name + " sm_" + std::to_string(prop.major) +
                        std::to_string(prop.minor));
    auto* c = new nomad_b200_ctx();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    NB_CUDA(cudaSetDevice(device));
    NB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    c->own_stream = true;
    *out = c;
  });
}

int32_t nomad_b200_destroy(nomad_b200_ctx* c) {
  return guard([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    nb::release_ring(c);  // waits for its own copies only
    if (c->own_stream && c->stream) {
      cudaStreamSynchronize(c->stream);
      cudaStreamDestroy(c->stream);
    }
    cudaGetLastError();  // teardown errors are not reported to later launches
    delete c;
  });
}

int32_t nomad_b200_set_stream(nomad_b200_ctx* c, void* s) {
  return guard([&] {
    if (!c) fail(kParameter, "ctx is NULL");
    bind_device(c);
    if (c->own_stream && c->stream) {
      NB_CUDA(cudaStreamSynchronize(c->stream));
      NB_CUDA(cudaStreamDestroy(c->stream));
    }
    if (s) {
      c->stream = static_cast<cudaStream_t>(s);
      c->own_stream = false;
    } else {
      NB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
  });
}

uint64_t nomad_b200_kernel_launches(const nomad_b200_ctx* c) { return c ? c->launches : 0; }

int32_t nomad_b200_nccl_unique_id(void* out128) {
  return guard([&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) fail(kInternal, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out128, &id, 128);
  });
}

static int32_t generate_mixture(nomad_b200_ctx* c, uint64_t row0, uint64_t rows, uint64_t dims,
                                uint64_t blobs, double spread, uint64_t seed, void* out,
                                bool bf16) {
  return guard([&] {
    if (!c || !out) fail(kParameter, "NULL argument");
    if (rows < 1 || dims < 1 || blobs < 1) fail(kParameter, "empty mixture shape");
    bind_device(c);
    DBuf<float> centres(blobs * dims + 4);
    const uint32_t s0 = (uint32_t)seed, s1 = (uint32_t)(seed >> 32) ^ 0x5eedu;
    const uint64_t cq = (blobs * dims + 3) / 4;
    k_mixture_centres<<<(unsigned)((cq + 255) / 256), 256, 0, c->stream>>>(
        centres.p, blobs * dims, (float)spread, s0, s1);
    note_launch(c, "k_mixture_centres");
    if (bf16)
      k_mixture_points<<<c->sm_count * 8, 256, 0, c->stream>>>(
          static_cast<__nv_bfloat16*>(out), centres.p, row0, rows, dims, blobs, s0, s1);
    else
      k_mixture_points<<<c->sm_count * 8, 256, 0, c->stream>>>(static_cast<float*>(out),
                                                               centres.p, row0, rows, dims, blobs,
                                                               s0, s1);
    note_launch(c, "k_mixture_points");
    NB_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int32_t nomad_b200_generate_mixture(nomad_b200_ctx* c, uint64_t rows, uint64_t dims,
                                    uint64_t blobs, double spread, uint64_t seed, float* out) {
  return generate_mixture(c, 0, rows, dims, blobs, spread, seed, out, false);
}

int32_t nomad_b200_generate_mixture_bf16(nomad_b200_ctx* c, uint64_t rows, uint64_t dims,
                                         uint64_t blobs, double spread, uint64_t seed,
                                         void* out) {
  return generate_mixture(c, 0, rows, dims, blobs, spread, seed, out, true);
}

int32_t nomad_b200_generate_mixture_rows(nomad_b200_ctx* c, uint64_t row0, uint64_t rows,
                                         uint64_t dims, uint64_t blobs, double spread,
                                         uint64_t seed, int32_t dtype, void* out) {
  return generate_mixture(c, row0, rows, dims, blobs, spread, seed, out, dtype == NOMAD_B200_BF16);
}

}  // extern "C"
