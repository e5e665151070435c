// Micro-benchmark: random 16-byte row updates, 2x RED.F64 vs one 16-B
// cp.reduce.async.bulk (UBLKRED.ADD.F64) vs non-atomic RMW, over a 20 MB
// (L2-resident) array.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 red_bench.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
__global__ void k_red(double2* p, uint32_t n, uint32_t per) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t i = 0; i < per; ++i) {
    uint32_t r = hsh(t * 7919u + i) % n;
    atomicAdd(&p[r].x, 1e-9);
    atomicAdd(&p[r].y, -1e-9);
  }
}
__global__ void k_bulk(double2* p, uint32_t n, uint32_t per) {
  __shared__ __align__(16) double2 s[256];
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  s[threadIdx.x] = make_double2(1e-9, -1e-9);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  unsigned sa = (unsigned)__cvta_generic_to_shared(&s[threadIdx.x]);
  for (uint32_t i = 0; i < per; ++i) {
    uint32_t r = hsh(t * 7919u + i) % n;
    asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 16;"
                 :: "l"(p + r), "r"(sa) : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__global__ void k_rmw(double2* p, uint32_t n, uint32_t per) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t i = 0; i < per; ++i) {
    uint32_t r = hsh(t * 7919u + i) % n;
    double2 v = p[r]; v.x += 1e-9; v.y -= 1e-9; p[r] = v;
  }
}
// double-float rows {hi.x, hi.y, lo.x, lo.y}: one RED.F32x2 onto lo
__global__ void k_red32x2(double2* p, uint32_t n, uint32_t per) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  float* f = reinterpret_cast<float*>(p);
  for (uint32_t i = 0; i < per; ++i) {
    uint32_t r = hsh(t * 7919u + i) % n;
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" :: "l"(f + 4 * (uint64_t)r + 2),
                 "f"(1e-9f), "f"(-1e-9f) : "memory");
  }
}
// one RED.F64 per row (x only): the per-instruction cost reference
__global__ void k_red1(double2* p, uint32_t n, uint32_t per) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t i = 0; i < per; ++i) {
    uint32_t r = hsh(t * 7919u + i) % n;
    atomicAdd(&p[r].x, 1e-9);
  }
}
// lane pairs (2i, 2i+1) add to x and y of the same row in one RED.F64
// instruction: 16 rows per warp instruction, half the instructions per row
__global__ void k_red_pair(double2* p, uint32_t n, uint32_t per) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  double* q = reinterpret_cast<double*>(p);
  for (uint32_t i = 0; i < per; ++i) {
    // 2 rows per thread-pair per iteration keeps the update count equal to k_red
    const uint32_t pair = (t >> 1);
    const uint32_t r0 = hsh(pair * 7919u + 2 * i) % n, r1 = hsh(pair * 7919u + 2 * i + 1) % n;
    atomicAdd(q + 2 * (uint64_t)r0 + (lane & 1), (lane & 1) ? -1e-9 : 1e-9);
    atomicAdd(q + 2 * (uint64_t)r1 + (lane & 1), (lane & 1) ? -1e-9 : 1e-9);
  }
}
int main() {
  const uint32_t n = 1250000;  // 20 MB of double2
  double2* p; cudaMalloc(&p, n * 16); cudaMemset(p, 0, n * 16);
  const uint32_t blocks = 148 * 8, threads = 256, per = 1400;  // ~424M row updates
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  const char* names[6] = {"2xRED.F64", "UBLKRED16", "RMW(non-atomic)", "1xRED.F32x2", "1xRED.F64",
                          "RED.F64 lane pairs"};
  for (int v = 0; v < 6; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (v == 0) k_red<<<blocks, threads>>>(p, n, per);
      if (v == 1) k_bulk<<<blocks, threads>>>(p, n, per);
      if (v == 2) k_rmw<<<blocks, threads>>>(p, n, per);
      if (v == 3) k_red32x2<<<blocks, threads>>>(p, n, per);
      if (v == 4) k_red1<<<blocks, threads>>>(p, n, per);
      if (v == 5) k_red_pair<<<blocks, threads>>>(p, n, per);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    }
    double upd = (double)blocks * threads * per;
    printf("%-16s %8.3f ms  %.1f G row-updates/s  err=%s\n", names[v], ms, upd / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
