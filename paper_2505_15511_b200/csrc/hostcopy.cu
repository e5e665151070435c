// Bulk copies between device memory and caller-owned host memory.
//
// The C-ABI hands results back into whatever host buffers the caller passes
// (numpy arrays, std::vectors: pageable, often freshly allocated). A pageable
// cudaMemcpy into a fresh buffer runs at the speed of one host thread taking
// the first-touch page faults: 3.9 GB/s measured on the B200 box for a
// 1.8 GB kNN graph (tools/d2h_probe.py), against 51.7 GB/s into pinned memory.
// Large copies therefore go through a pinned two-buffer ring owned by the
// context: the DMA of chunk i+1 overlaps the host-side copy of chunk i, and
// the host side is split over several threads so the page faults are taken
// in parallel. Pinned / registered destinations are copied directly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"
#include "hostcopy.cuh"

namespace nb {
namespace {

constexpr size_t kChunk = 64ull << 20;     // bytes per staging buffer
constexpr size_t kDirect = 8ull << 20;     // below this: one plain copy
constexpr size_t kSlice = 4ull << 20;      // min bytes per host thread

bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void par_memcpy(void* dst, const void* src, size_t bytes) {
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t T = std::min<size_t>({(size_t)8, (size_t)hw, std::max<size_t>(1, bytes / kSlice)});
  if (T <= 1) {
    std::memcpy(dst, src, bytes);
    return;
  }
  const size_t per = ((bytes + T - 1) / T + 4095) & ~size_t(4095);  // page-aligned slices
  std::vector<std::thread> th;
  th.reserve(T);
  for (size_t t = 0; t < T; ++t) {
    const size_t a = t * per;
    if (a >= bytes) break;
    const size_t n = std::min(per, bytes - a);
    th.emplace_back([=] { std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, n); });
  }
  for (auto& x : th) x.join();
}

void ensure_ring(nomad_b200_ctx* c) {
  if (c->pin[0]) return;
  for (int b = 0; b < 2; ++b) {
    NB_CUDA(cudaMallocHost(&c->pin[b], kChunk));
    NB_CUDA(cudaEventCreateWithFlags(&c->pin_ev[b], cudaEventDisableTiming));
  }
}

}  // namespace

void copy_d2h(nomad_b200_ctx* c, void* dst, const void* src, size_t bytes) {
  cudaStream_t S = c->stream;
  if (!bytes) return;
  if (bytes < kDirect || is_pinned(dst)) {
    NB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    return;
  }
  ensure_ring(c);
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](size_t i) {
    const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
    NB_CUDA(cudaMemcpyAsync(c->pin[i & 1], static_cast<const char*>(src) + off, n,
                            cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaEventRecord(c->pin_ev[i & 1], S));
  };
  issue(0);
  for (size_t i = 0; i < nch; ++i) {
    // buffer (i+1)&1 was drained by the host copy of chunk i-1 (synchronous)
    if (i + 1 < nch) issue(i + 1);
    NB_CUDA(cudaEventSynchronize(c->pin_ev[i & 1]));
    const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
    par_memcpy(static_cast<char*>(dst) + off, c->pin[i & 1], n);
  }
}

void copy_h2d(nomad_b200_ctx* c, void* dst, const void* src, size_t bytes) {
  cudaStream_t S = c->stream;
  if (!bytes) return;
  if (bytes < kDirect || is_pinned(src)) {
    NB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, S));
    NB_CUDA(cudaStreamSynchronize(S));
    return;
  }
  ensure_ring(c);
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  bool used[2] = {false, false};
  for (size_t i = 0; i < nch; ++i) {
    const int b = (int)(i & 1);
    if (used[b]) NB_CUDA(cudaEventSynchronize(c->pin_ev[b]));  // its previous DMA is done
    const size_t off = i * kChunk, n = std::min(kChunk, bytes - off);
    par_memcpy(c->pin[b], static_cast<const char*>(src) + off, n);
    NB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, c->pin[b], n, cudaMemcpyHostToDevice, S));
    NB_CUDA(cudaEventRecord(c->pin_ev[b], S));
    used[b] = true;
  }
  NB_CUDA(cudaStreamSynchronize(S));
}

void copy_out(nomad_b200_ctx* c, void* dst, const void* src, size_t bytes, bool dst_on_device) {
  if (dst_on_device) {
    NB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, c->stream));
    NB_CUDA(cudaStreamSynchronize(c->stream));
  } else {
    copy_d2h(c, dst, src, bytes);
  }
}

void release_ring(nomad_b200_ctx* c) {
  for (int b = 0; b < 2; ++b) {
    if (c->pin_ev[b]) {
      cudaEventSynchronize(c->pin_ev[b]);
      cudaEventDestroy(c->pin_ev[b]);
      c->pin_ev[b] = nullptr;
    }
    if (c->pin[b]) {
      cudaFreeHost(c->pin[b]);
      c->pin[b] = nullptr;
    }
  }
}

}  // namespace nb
