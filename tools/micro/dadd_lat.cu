// Dependent-chain latency of fp64 add (no FMA contraction) and of the
// smem-load -> widen -> add step of the sequential column sums, in SM cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dadd_lat dadd_lat.cu && ./dadd_lat
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dadd(double* out, double a, int n, long long* cyc) {
  double acc = a;
  const double b = a * 1e-3;
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, b);
  const long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

__global__ void k_lds_dadd(double* out, int n, long long* cyc) {
  __shared__ float s[256 * 33];
  for (int i = threadIdx.x; i < 256 * 33; i += blockDim.x) s[i] = 1.0f + i * 1e-7f;
  __syncthreads();
  double acc = 0.0;
  const int lane = threadIdx.x & 31;
  const long long t0 = clock64();
  for (int rep = 0; rep < n / 256; ++rep)
    for (int r = 0; r < 256; ++r) acc = __dadd_rn(acc, (double)s[r * 33 + lane]);
  const long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaMallocManaged(&cyc, sizeof(long long));
  const int n = 1 << 20;
  k_dadd<<<1, 32>>>(out, 1.0, n, cyc);
  cudaDeviceSynchronize();
  k_dadd<<<1, 32>>>(out, 1.0, n, cyc);
  cudaDeviceSynchronize();
  printf("dependent DADD chain: %.2f cycles per add\n", (double)*cyc / n);
  k_lds_dadd<<<1, 32>>>(out, n, cyc);
  cudaDeviceSynchronize();
  k_lds_dadd<<<1, 32>>>(out, n, cyc);
  cudaDeviceSynchronize();
  printf("LDS + F2F.F64.F32 + dependent DADD (column-sum step): %.2f cycles per row\n",
         (double)*cyc / n);
  return 0;
}
