// Does separating the SGD kernel's gathers and REDs in time (whole-GPU phases
// with a grid barrier) beat the mixed L2 request rate? Same per-thread work
// as mix_bench's k_mix (8 gathers + 14 lane-pair REDs per iteration, 20 MB
// L2-resident array), gathers of B iterations, grid.sync(), REDs of B
// iterations, grid.sync(), ...
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 phase_bench.cu -o phase_bench
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

__global__ void __launch_bounds__(256) k_phase(double2* p, uint32_t n, uint32_t per, uint32_t B,
                                               double* sink) {
  cg::grid_group g = cg::this_grid();
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  double* q = reinterpret_cast<double*>(p);
  double acc = 0.0;
  for (uint32_t i0 = 0; i0 < per; i0 += B) {
    const uint32_t i1 = min(per, i0 + B);
    for (uint32_t i = i0; i < i1; ++i) {
      double2 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __ldcg(p + hsh(t * 7919u + 64 * i + j) % n);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += v[j].x + v[j].y;
    }
    if (B < per) g.sync();
    for (uint32_t i = i0; i < i1; ++i) {
#pragma unroll
      for (int j = 0; j < 14; ++j) {
        const uint32_t r = hsh((t >> 1) * 104729u + 64 * i + 16 + j) % n;
        atomicAdd(q + 2 * (uint64_t)r + (lane & 1), (lane & 1) ? -1e-12 : 1e-12);
      }
    }
    if (B < per) g.sync();
  }
  if (acc == 12345.678) sink[t] = acc;
}

int main() {
  const uint32_t n = 1250000;
  double2* p;
  double* sink;
  cudaMalloc(&p, n * 16);
  cudaMemset(p, 0, n * 16);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_phase, 256, 0);
  const uint32_t blocks = 148 * per_sm;
  cudaMalloc(&sink, (size_t)blocks * 256 * 8);
  const uint32_t per = 100 * 8 / per_sm;  // same total work as mix_bench at 8 blocks/SM
  printf("resident blocks/SM %d\n", per_sm);
  for (uint32_t B : {1u, 2u, 4u, 8u, 16u, 1000u}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0.f;
    uint32_t nn = n, pp = per, BB = B;
    void* args[] = {&p, &nn, &pp, &BB, &sink};
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k_phase, blocks, 256, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double req = (double)blocks * 256 * per * (8 + 7);
    printf("phase B=%4u iterations  %7.3f ms  %6.1f G req/s  (10M-head epoch %.3f ms)  %s\n", B, ms,
           req / ms / 1e6, 10e6 * 45 / (req / ms), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
