// Request-mix sweep for the throughput SGD kernel's binding unit: 16-byte row
// gathers mixed 24:21 (requests) with lane-pair RED.F64 row updates on an
// L2-resident 20 MB double2 array, varying
//   - the load flavour (L1-allocating ld, ld.cg, ld.nc, ld with L1::no_allocate),
//   - the issue order (all gathers then all REDs, or interleaved),
//   - resident warps per SM (blocks of 256 threads per SM),
// to see whether the mixed rate is an L2 limit or an SM-side (occupancy /
// outstanding-request) limit.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mix_bench.cu -o mix_bench
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int LK>
__device__ __forceinline__ double2 ld(const double2* p) {
  double2 v;
  if constexpr (LK == 0) {
    v = *p;
  } else if constexpr (LK == 1) {
    v = __ldcg(p);
  } else if constexpr (LK == 2) {
    v = __ldg(p);
  } else {
    asm volatile("ld.global.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  }
  return v;
}

// per iteration: 8 gather instructions (256 requests / warp) and 14 lane-pair
// RED instructions (224 requests / warp) = the 24:21 per-head request mix
template <int LK, bool INTER>
__global__ void __launch_bounds__(256) k_mix(double2* p, uint32_t n, uint32_t per, double* sink) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  double* q = reinterpret_cast<double*>(p);
  double acc = 0.0;
  for (uint32_t i = 0; i < per; ++i) {
    double2 v[8];
    if constexpr (INTER) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[j] = ld<LK>(p + hsh(t * 7919u + 64 * i + j) % n);
        const uint32_t r = hsh((t >> 1) * 104729u + 64 * i + 16 + j) % n;
        atomicAdd(q + 2 * (uint64_t)r + (lane & 1), (lane & 1) ? -1e-12 : 1e-12);
      }
#pragma unroll
      for (int j = 8; j < 14; ++j) {
        const uint32_t r = hsh((t >> 1) * 104729u + 64 * i + 16 + j) % n;
        atomicAdd(q + 2 * (uint64_t)r + (lane & 1), (lane & 1) ? -1e-12 : 1e-12);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = ld<LK>(p + hsh(t * 7919u + 64 * i + j) % n);
#pragma unroll
      for (int j = 0; j < 14; ++j) {
        const uint32_t r = hsh((t >> 1) * 104729u + 64 * i + 16 + j) % n;
        atomicAdd(q + 2 * (uint64_t)r + (lane & 1), (lane & 1) ? -1e-12 : 1e-12);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j].x + v[j].y;
  }
  if (acc == 12345.678) sink[t] = acc;
}

template <int LK>
__global__ void __launch_bounds__(256) k_gather(const double2* p, uint32_t n, uint32_t per, double* sink) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (uint32_t i = 0; i < per; i += 8) {
    double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = ld<LK>(p + hsh(t * 7919u + i + j) % n);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j].x + v[j].y;
  }
  if (acc == 12345.678) sink[t] = acc;
}

static const char* LKN[4] = {"ld (L1 alloc)", "ld.cg", "ld.nc", "ld.L1::no_allocate"};

template <int LK, bool INTER>
static void mix(double2* p, uint32_t n, double* sink, int bps) {
  const uint32_t blocks = 148 * bps;
  // same total work for every occupancy: 148*8 blocks x 100 iterations
  const uint32_t per = 100 * 8 / bps;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0.f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_mix<LK, INTER><<<blocks, 256>>>(p, n, per, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  const double req = (double)blocks * 256 * per * (8 + 7);
  printf("mix %-20s %-11s warps/SM %2d  %7.3f ms  %6.1f G req/s  (10M-head epoch floor %.3f ms) %s\n",
         LKN[LK], INTER ? "interleaved" : "blocked", bps * 8, ms, req / ms / 1e6,
         10e6 * 45 / (req / ms) , cudaGetErrorString(cudaGetLastError()));
}

template <int LK>
static void gather(double2* p, uint32_t n, double* sink, int bps) {
  const uint32_t blocks = 148 * bps;
  const uint32_t per = 1408 * 8 / bps;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0.f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_gather<LK><<<blocks, 256>>>(p, n, per, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  const double req = (double)blocks * 256 * per;
  printf("gather %-20s warps/SM %2d  %7.3f ms  %6.1f G req/s %s\n", LKN[LK], bps * 8, ms,
         req / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const uint32_t n = 1250000;  // 20 MB of double2 (one config-C shard)
  double2* p;
  double* sink;
  cudaMalloc(&p, n * 16);
  cudaMemset(p, 0, n * 16);
  cudaMalloc(&sink, 148 * 8 * 256 * 8);
  for (int bps : {2, 3, 4, 8}) {
    gather<0>(p, n, sink, bps);
    gather<1>(p, n, sink, bps);
    gather<2>(p, n, sink, bps);
  }
  for (int bps : {2, 3, 4, 8}) {
    mix<0, false>(p, n, sink, bps);
    mix<1, false>(p, n, sink, bps);
    mix<2, false>(p, n, sink, bps);
    mix<3, false>(p, n, sink, bps);
    mix<0, true>(p, n, sink, bps);
    mix<2, true>(p, n, sink, bps);
  }
  return 0;
}
