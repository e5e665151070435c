// Micro-benchmark for the SGD kernel's binding unit:
//  1. random 16-byte row gathers from an L2-resident 20 MB double2 array;
//  2. gathers mixed 24:21 (requests) with lane-pair RED.F64 row updates,
//     the per-head request mix of k_sgd_hogwild;
//  3. the same row updates / gathers against distributed shared memory of a
//     thread-block cluster (rows resident in the cluster's shared memory):
//     red.shared::cluster.add.f64 lane pairs and ld.shared::cluster.v2.f64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 gather_bench.cu -o gather_bench
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// 8 independent random row loads per iteration per lane
__global__ void k_gather(const double2* __restrict__ p, uint32_t n, uint32_t per, double* sink) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (uint32_t i = 0; i < per; i += 8) {
    double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcg(p + hsh(t * 7919u + i + j) % n);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j].x + v[j].y;
  }
  if (acc == 12345.678) sink[t] = acc;
}

// per iteration: 8 gather instructions (256 requests / warp) and 14 lane-pair
// RED instructions (224 requests / warp) = the 24:21 per-head request mix
__global__ void k_mix(double2* p, uint32_t n, uint32_t per, double* sink) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  double* q = reinterpret_cast<double*>(p);
  double acc = 0.0;
  for (uint32_t i = 0; i < per; ++i) {
    double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcg(p + hsh(t * 7919u + 64 * i + j) % n);
#pragma unroll
    for (int j = 0; j < 14; ++j) {
      const uint32_t r = hsh((t >> 1) * 104729u + 64 * i + 16 + j) % n;
      atomicAdd(q + 2 * (uint64_t)r + (lane & 1), (lane & 1) ? -1e-12 : 1e-12);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j].x + v[j].y;
  }
  if (acc == 12345.678) sink[t] = acc;
}

// lane-pair REDs only (the round-1 reference rate)
__global__ void k_red_pair(double2* p, uint32_t n, uint32_t per) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  double* q = reinterpret_cast<double*>(p);
  for (uint32_t i = 0; i < per; ++i) {
    const uint32_t r = hsh((t >> 1) * 7919u + i) % n;
    atomicAdd(q + 2 * (uint64_t)r + (lane & 1), (lane & 1) ? -1e-12 : 1e-12);
  }
}

// DSMEM: each CTA of a cluster holds `rows` double2 rows in shared memory;
// lanes update / read random rows anywhere in the cluster.
template <int MODE>  // 0: lane-pair remote RED.F64, 1: remote 16-B loads, 2: local-CTA RED
__global__ void k_dsmem(uint32_t rows, uint32_t per, double* sink) {
  extern __shared__ __align__(16) double2 srow[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t csz = cl.num_blocks();
  for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) srow[i] = make_double2(0.0, 0.0);
  cl.sync();
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(srow);
  double acc = 0.0;
  for (uint32_t i = 0; i < per; ++i) {
    const uint32_t h = hsh(((MODE == 1 ? t : (t >> 1))) * 7919u + i);
    const uint32_t cta = MODE == 2 ? cl.block_rank() : h % csz;
    const uint32_t r = (h / csz) % rows;
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base + 16 * r), "r"(cta));
    if (MODE == 1) {
      double a, b;
      asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(ra));
      acc += a + b;
    } else {
      asm volatile("red.shared::cluster.add.f64 [%0], %1;" ::"r"(ra + 8 * (lane & 1)),
                   "d"((lane & 1) ? -1e-12 : 1e-12)
                   : "memory");
    }
  }
  cl.sync();
  if (acc == 12345.678) sink[t] = acc;
}

template <int MODE>
static float run_dsmem(int csz, uint32_t rows, uint32_t per, double* sink, int* nclusters) {
  const size_t smem = (size_t)rows * 16;
  auto kern = k_dsmem<MODE>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csz;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int maxc = 0;
  cfg.gridDim = dim3(csz);
  cudaOccupancyMaxActiveClusters(&maxc, kern, &cfg);
  *nclusters = maxc;
  cfg.gridDim = dim3(csz * (maxc > 0 ? maxc : 1));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0.f;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    cudaLaunchKernelEx(&cfg, kern, rows, per, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
  }
  return ms;
}

int main() {
  const uint32_t n = 1250000;  // 20 MB of double2 (one config-C shard)
  double2* p;
  double* sink;
  cudaMalloc(&p, n * 16);
  cudaMemset(p, 0, n * 16);
  cudaMalloc(&sink, 148 * 8 * 512 * 8);
  const uint32_t blocks = 148 * 8, threads = 256;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms = 0.f;
  // 1. gathers
  {
    const uint32_t per = 1408;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k_gather<<<blocks, threads>>>(p, n, per, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double req = (double)blocks * threads * per;
    printf("gather 16B rows (L2-resident 20 MB)      %8.3f ms  %6.1f G requests/s  err=%s\n", ms,
           req / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  // 2. lane-pair REDs alone
  {
    const uint32_t per = 1400;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k_red_pair<<<blocks, threads>>>(p, n, per);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double req = (double)blocks * threads * per / 2;  // two lanes per request
    printf("lane-pair RED.F64 row updates            %8.3f ms  %6.1f G requests/s  err=%s\n", ms,
           req / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  // 3. the 24:21 mix
  {
    const uint32_t per = 100;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k_mix<<<blocks, threads>>>(p, n, per, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double req = (double)blocks * threads * per * (8 + 7);  // 8 loads + 14/2 pair requests
    printf("mix 24:21 gathers : pair-RED requests    %8.3f ms  %6.1f G requests/s  err=%s\n", ms,
           req / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    printf("  => per 10M-head epoch at 45 requests/head: %.3f ms floor\n", 10e6 * 45 / (req / ms));
  }
  // 4. distributed shared memory
  const int sizes[3] = {16, 8, 2};
  for (int si = 0; si < 3; ++si) {
    const int csz = sizes[si];
    const uint32_t rows = 12800;  // 200 KB per CTA
    const uint32_t per = 2000;
    int ncl = 0;
    float m0 = run_dsmem<0>(csz, rows, per, sink, &ncl);
    const char* e0 = cudaGetErrorString(cudaGetLastError());
    float m1 = run_dsmem<1>(csz, rows, per, sink, &ncl);
    const char* e1 = cudaGetErrorString(cudaGetLastError());
    float m2 = run_dsmem<2>(csz, rows, per, sink, &ncl);
    const char* e2 = cudaGetErrorString(cudaGetLastError());
    const double lanes = (double)csz * ncl * 512 * per;
    printf("DSMEM cluster %2d (%3d clusters resident, %u rows/CTA): remote pair-RED %6.1f G rows/s (%s)"
           "  remote ld.v2.f64 %6.1f G rows/s (%s)  local-CTA pair-RED %6.1f G rows/s (%s)\n",
           csz, ncl, rows, lanes / 2 / m0 / 1e6, e0, lanes / m1 / 1e6, e1, lanes / 2 / m2 / 1e6, e2);
  }
  return 0;
}
