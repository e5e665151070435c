// Bulk device <-> caller-host copies through the context's pinned staging
// ring (hostcopy.cu). All are ordered after the work already on ctx->stream
// and return when the data has arrived.
#pragma once
#include <cstddef>

struct nomad_b200_ctx;

namespace nb {
void copy_d2h(nomad_b200_ctx* c, void* dst_host, const void* src_dev, size_t bytes);
void copy_h2d(nomad_b200_ctx* c, void* dst_dev, const void* src_host, size_t bytes);
// dst on the device (one device copy) or in host memory (copy_d2h)
void copy_out(nomad_b200_ctx* c, void* dst, const void* src_dev, size_t bytes, bool dst_on_device);
void release_ring(nomad_b200_ctx* c);
}  // namespace nb
