// Can whole-GPU gather / RED phases be aligned by the global timer instead of
// a grid barrier? Same per-thread work as mix_bench's k_mix iteration (8
// gathers, then 14 lane-pair REDs), but every thread starts its gathers at a
// window boundary of %globaltimer and its REDs Wg ns later; windows repeat
// every Wg + Wr ns. 20 MB L2-resident array, 8 blocks/SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 window_bench.cu -o window_bench
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(256) k_window(double2* p, uint32_t n, uint32_t per, uint32_t wg,
                                                uint32_t wr, double* sink) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  double* q = reinterpret_cast<double*>(p);
  double acc = 0.0;
  const uint64_t period = (uint64_t)wg + wr;
  uint64_t w = (gtime() / period + 2) * period;  // common window grid (global time)
  for (uint32_t i = 0; i < per; ++i) {
    if (period) while (gtime() < w) {}
    double2 v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = __ldcg(p + hsh(t * 7919u + 64 * i + j) % n);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j].x + v[j].y;
    if (period) while (gtime() < w + wg) {}
#pragma unroll
    for (int j = 0; j < 14; ++j) {
      const uint32_t r = hsh((t >> 1) * 104729u + 64 * i + 16 + j) % n;
      atomicAdd(q + 2 * (uint64_t)r + (lane & 1), (lane & 1) ? -1e-12 : 1e-12);
    }
    w += period;
  }
  if (acc == 12345.678) sink[t] = acc;
}

int main() {
  const uint32_t n = 1250000;
  double2* p;
  double* sink;
  cudaMalloc(&p, n * 16);
  cudaMemset(p, 0, n * 16);
  const uint32_t blocks = 148 * 8;
  cudaMalloc(&sink, (size_t)blocks * 256 * 8);
  const uint32_t per = 100;
  struct W { uint32_t g, r; } ws[] = {{0, 0},       {6000, 9000},   {8000, 11000}, {9000, 12000},
                                      {10000, 14000}, {12000, 16000}, {14000, 18000}};
  for (auto x : ws) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float ms = 0.f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      k_window<<<blocks, 256>>>(p, n, per, x.g, x.r, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
    }
    const double req = (double)blocks * 256 * per * (8 + 7);
    printf("windows gather %5u ns / red %5u ns  %7.3f ms  %6.1f G req/s  (10M-head epoch %.3f ms) %s\n",
           x.g, x.r, ms, req / ms / 1e6, 10e6 * 45 / (req / ms), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
