// Shared host/device plumbing for libnomad_b200.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "nomad_b200.h"

namespace nb {

// ErrorKind order of error.hpp:25-36; status = 1 + kind.
enum Kind { kIo = 0, kDimension, kValidation, kSchema, kParameter, kConfig,
            kDegenerate, kDivergence, kSize, kInternal };

struct Error : std::runtime_error {
  Kind kind;
  Error(Kind k, const std::string& m) : std::runtime_error(m), kind(k) {}
};

[[noreturn]] inline void fail(Kind k, const std::string& m) { throw Error(k, m); }

void set_last_error(const std::string& m);

#define NB_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      ::nb::fail(::nb::kInternal, std::string("CUDA error ") +               \
                                      cudaGetErrorString(e_) + " at " +      \
                                      __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// C-ABI wrapper: runs f, maps exceptions to status codes.
template <class F>
int32_t guard(F&& f) {
  try {
    f();
    return NOMAD_B200_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    cudaGetLastError();  // a reported CUDA error must not resurface at a later launch
    return 1 + static_cast<int32_t>(e.kind);
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return NOMAD_B200_ERR_INTERNAL;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return NOMAD_B200_ERR_INTERNAL;
  }
}

// Large device blocks (>= 64 MB) are recycled instead of returned to the
// driver: cudaMalloc / cudaFree of GB-sized blocks occasionally stall for
// hundreds of ms (mapping / unmapping), which made the index build's
// per-cluster stages jittery. A released block is kept only after a device
// synchronisation (the semantics cudaFree had), so reuse is race-free; the
// cache is bounded and flushed when an allocation runs out of memory.
void* dev_alloc(size_t bytes);
void dev_free(void* p, size_t bytes);

// RAII device buffer on the current device.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
  }
  void release() {
    if (p) dev_free(p, n * sizeof(T));
    p = nullptr;
    n = 0;
  }
  size_t bytes() const { return n * sizeof(T); }
};

}  // namespace nb

// The opaque context of the C-ABI.
struct nomad_b200_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint64_t launches = 0;
  int sm_count = 148;
  // statistics of the last build_knn call
  uint64_t knn_tc_uncertified = 0, knn_exhaustive = 0, knn_sub_certified = 0;
  // pinned staging ring for bulk copies to / from caller host memory (hostcopy.cu)
  void* pin[2] = {nullptr, nullptr};
  cudaEvent_t pin_ev[2] = {nullptr, nullptr};
};

// A set of contexts driven by one host thread (nomad_b200_group_create):
// distinct devices joined by NCCL communicators, or G contexts on one device
// sharing one stream (loopback exchange).
struct nomad_b200_group {
  std::vector<nomad_b200_ctx*> ctx;  // owned, one per rank
  std::vector<void*> comm;           // ncclComm_t per rank (distinct devices), else empty
  bool loopback = false;
};

namespace nb {
// Makes ctx's device current for this host thread.
void bind_device(nomad_b200_ctx* c);
// Launch bookkeeping: every kernel launch goes through this so the context can
// report how many of its kernels ran (gpu_launches evidence) and surface
// launch-configuration errors immediately.
void note_launch(nomad_b200_ctx* c, const char* name);
}  // namespace nb
