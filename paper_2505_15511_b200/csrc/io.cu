// Data I/O at the path's two ends: the raw-f32 vector
// loader streaming straight into device memory (dataset.hpp:122-173) and the
// layout writers — the reference's `id,x,y[,label]` CSV with %.17g
// (dataset.hpp:223-250), formatted on all host cores, and a raw f64 dump.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "index_common.cuh"

namespace nb {

namespace {

// First non-finite value (row-major index) of a device chunk.
__global__ void k_first_nonfinite(const float* v, uint64_t count, uint64_t base,
                                  unsigned long long* first) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (!isfinite(v[i])) atomicMin(first, (unsigned long long)(base + i));
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

void shape_from_size(const std::string& path, uint64_t bytes, uint64_t& n, uint64_t& d) {
  // dataset.hpp:131-152
  if (!n && !d) fail(kParameter, "raw-f32 needs --rows and/or --dims");
  if (bytes % 4 != 0)
    fail(kDimension, "file size " + std::to_string(bytes) + " is not a multiple of 4 bytes");
  const uint64_t values = bytes / 4;
  if (n && d) {
    if (n * d != values)
      fail(kDimension, "file holds " + std::to_string(bytes) + " bytes but rows*dims*4 = " +
                           std::to_string(n * d * 4));
  } else if (n) {
    if (values % n != 0) fail(kDimension, "file size not divisible by rows");
    d = values / n;
  } else {
    if (values % d != 0) fail(kDimension, "file size not divisible by dims");
    n = values / d;
  }
  (void)path;
}

[[noreturn]] void nonfinite(uint64_t idx, uint64_t d) {
  fail(kValidation, "non-finite value at row " + std::to_string(idx / d) + ", column " +
                        std::to_string(idx % d));
}

}  // namespace

// The reference's save_layout byte for byte (ids NULL -> "0".."n-1", the
// default ids of the raw loader, dataset.hpp:79-82).
void save_layout_csv(const char* path, const double* lay, uint64_t n, const char* const* ids,
                     const char* const* labels) {
  File out;
  out.f = std::fopen(path, "wb");
  if (!out.f) fail(kIo, std::string("cannot write '") + path + "'");
  const bool with_labels = labels != nullptr;
  const char* hdr = with_labels ? "id,x,y,label\n" : "id,x,y\n";
  if (std::fputs(hdr, out.f) < 0) fail(kIo, std::string("write failed on '") + path + "'");
  const uint64_t block = 1 << 16;
  const unsigned T = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::string> part(T);
  for (uint64_t r0 = 0; r0 < n; r0 += block * T) {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; ++t) {
      th.emplace_back([&, t] {
        std::string& s = part[t];
        s.clear();
        const uint64_t a = r0 + t * block, b = std::min(n, a + block);
        char buf[96];
        for (uint64_t i = a; i < b; ++i) {
          if (ids) s += ids[i]; else s += std::to_string(i);
          std::snprintf(buf, sizeof buf, ",%.17g,%.17g", lay[2 * i], lay[2 * i + 1]);
          s += buf;
          if (with_labels) {
            s += ',';
            s += labels[i];
          }
          s += '\n';
        }
      });
    }
    for (auto& x : th) x.join();
    for (unsigned t = 0; t < T; ++t)
      if (!part[t].empty() && std::fwrite(part[t].data(), 1, part[t].size(), out.f) != part[t].size())
        fail(kIo, std::string("write failed on '") + path + "'");
  }
  if (std::fflush(out.f) != 0) fail(kIo, std::string("write failed on '") + path + "'");
}

}  // namespace nb

using namespace nb;

extern "C" {

int32_t nomad_b200_load_vectors_raw(nomad_b200_ctx* ctx, const char* path, uint64_t rows,
                                    uint64_t dims, float* out, int32_t out_location,
                                    uint64_t* rows_out, uint64_t* dims_out) {
  return guard([&] {
    if (!path) fail(kParameter, "NULL path");
    File in;
    in.f = std::fopen(path, "rb");
    if (!in.f) fail(kIo, std::string("cannot open '") + path + "'");
    if (std::fseek(in.f, 0, SEEK_END) != 0) fail(kIo, std::string("cannot seek '") + path + "'");
    const long long sz = std::ftell(in.f);
    if (sz < 0) fail(kIo, std::string("cannot size '") + path + "'");
    std::fseek(in.f, 0, SEEK_SET);
    uint64_t n = rows, d = dims;
    shape_from_size(path, (uint64_t)sz, n, d);
    // check_dataset_shape (dataset.hpp:84-87)
    if (n < 2) fail(kParameter, "dataset needs at least 2 rows");
    if (d < 1) fail(kParameter, "dataset needs at least 1 column");
    if (rows_out) *rows_out = n;
    if (dims_out) *dims_out = d;
    if (!out) return;  // shape query
    static_assert(sizeof(float) == 4, "f32");
    const uint32_t probe = 1;
    if (*reinterpret_cast<const uint8_t*>(&probe) != 1) fail(kInternal, "big-endian host");
    const uint64_t values = n * d;
    if (out_location != NOMAD_B200_DEVICE) {
      if (values && std::fread(out, 4, values, in.f) != values)
        fail(kIo, std::string("short read on '") + path + "'");
      for (uint64_t i = 0; i < values; ++i)
        if (!std::isfinite(out[i])) nonfinite(i, d);
      return;
    }
    // device: 64 MB pinned double buffer, copies overlap the next read
    if (!ctx) fail(kParameter, "device output needs a context");
    bind_device(ctx);
    cudaStream_t S = ctx->stream;
    const uint64_t CH = 16ull << 20;  // floats per chunk
    float* pin[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    DBuf<unsigned long long> first(1);
    NB_CUDA(cudaMemsetAsync(first.p, 0xFF, 8, S));
    struct Pinned {
      float** p;
      cudaEvent_t* e;
      ~Pinned() {
        for (int b = 0; b < 2; ++b) {
          if (e[b]) { cudaEventSynchronize(e[b]); cudaEventDestroy(e[b]); }
          if (p[b]) cudaFreeHost(p[b]);
        }
      }
    } guard_pin{pin, done};
    for (int b = 0; b < 2; ++b) {
      NB_CUDA(cudaMallocHost(&pin[b], std::min(CH, std::max<uint64_t>(values, 1)) * 4));
      NB_CUDA(cudaEventCreateWithFlags(&done[b], cudaEventDisableTiming));
    }
    uint64_t chunk = 0;
    for (uint64_t v0 = 0; v0 < values; v0 += CH, ++chunk) {
      const int b = (int)(chunk & 1);
      const uint64_t c = std::min(CH, values - v0);
      NB_CUDA(cudaEventSynchronize(done[b]));  // buffer b's previous copy finished
      if (std::fread(pin[b], 4, c, in.f) != c) fail(kIo, std::string("short read on '") + path + "'");
      NB_CUDA(cudaMemcpyAsync(out + v0, pin[b], c * 4, cudaMemcpyHostToDevice, S));
      NB_CUDA(cudaEventRecord(done[b], S));
      k_first_nonfinite<<<(unsigned)std::min<uint64_t>((c + 255) / 256, 4u * ctx->sm_count), 256, 0,
                          S>>>(out + v0, c, v0, first.p);
      note_launch(ctx, "k_first_nonfinite");
    }
    unsigned long long f = 0;
    NB_CUDA(cudaMemcpyAsync(&f, first.p, 8, cudaMemcpyDeviceToHost, S));
    NB_CUDA(cudaStreamSynchronize(S));
    if (f != ~0ull) nonfinite(f, d);
  });
}

int32_t nomad_b200_save_layout_csv(const char* path, const double* layout, uint64_t rows,
                                   const char* const* ids, const char* const* labels) {
  return guard([&] {
    if (!path || (!layout && rows)) fail(kParameter, "NULL argument");
    save_layout_csv(path, layout, rows, ids, labels);
  });
}

int32_t nomad_b200_save_layout_f64(const char* path, const double* layout, uint64_t rows) {
  return guard([&] {
    if (!path || (!layout && rows)) fail(kParameter, "NULL argument");
    File out;
    out.f = std::fopen(path, "wb");
    if (!out.f) fail(kIo, std::string("cannot write '") + path + "'");
    if (rows && std::fwrite(layout, 16, rows, out.f) != rows)
      fail(kIo, std::string("write failed on '") + path + "'");
    if (std::fflush(out.f) != 0) fail(kIo, std::string("write failed on '") + path + "'");
  });
}

}  // extern "C"
