// Multi-device group: the one-process form of the reference's W workers
// (optimizer.hpp:327-328, :399-408). One context per rank; distinct devices
// get one NCCL communicator each (ncclCommInitAll, single process), a list of
// one repeated device gets G contexts on one shared stream and a loopback
// exchange (device copies), so the G-rank math runs on one GPU.
#include <nccl.h>

#include <algorithm>
#include <set>

#include "common.cuh"

using namespace nb;

static void group_free(nomad_b200_group* g) {
  for (void* c : g->comm)
    if (c) ncclCommDestroy(static_cast<ncclComm_t>(c));
  g->comm.clear();
  // loopback: ranks > 0 borrow rank 0's stream, so they go first
  for (size_t r = g->ctx.size(); r-- > 0;)
    if (g->ctx[r]) nomad_b200_destroy(g->ctx[r]);
  g->ctx.clear();
  delete g;
}

extern "C" {

int32_t nomad_b200_group_create(const int32_t* devices, int32_t n, nomad_b200_group** out) {
  return guard([&] {
    if (!devices || !out) fail(kParameter, "NULL argument");
    if (n < 1) fail(kParameter, "a group needs at least one device");
    const std::set<int32_t> uniq(devices, devices + n);
    const bool loop = n > 1 && uniq.size() == 1;
    if (n > 1 && !loop && (int32_t)uniq.size() != n)
      fail(kParameter, "group devices must be all distinct (NCCL) or all the same (loopback)");
    auto* g = new nomad_b200_group();
    g->loopback = loop;
    try {
      for (int32_t r = 0; r < n; ++r) {
        nomad_b200_ctx* c = nullptr;
        if (nomad_b200_create(devices[r], &c) != NOMAD_B200_OK)
          fail(kInternal, std::string("group context: ") + nomad_b200_last_error());
        g->ctx.push_back(c);
        if (loop && r > 0) {  // one stream: program order is the exchange's ordering
          NB_CUDA(cudaSetDevice(c->device));
          NB_CUDA(cudaStreamDestroy(c->stream));
          c->stream = g->ctx[0]->stream;
          c->own_stream = false;
        }
      }
      if (n > 1 && !loop) {
        std::vector<ncclComm_t> comms(n);
        std::vector<int> devs(devices, devices + n);
        ncclResult_t r = ncclCommInitAll(comms.data(), n, devs.data());
        if (r != ncclSuccess) fail(kInternal, std::string("ncclCommInitAll: ") + ncclGetErrorString(r));
        for (auto c : comms) g->comm.push_back(c);
      }
    } catch (...) {
      group_free(g);
      throw;
    }
    *out = g;
  });
}

int32_t nomad_b200_group_destroy(nomad_b200_group* g) {
  return guard([&] {
    if (g) group_free(g);
  });
}

int32_t nomad_b200_group_size(const nomad_b200_group* g, int32_t* size, int32_t* loopback) {
  return guard([&] {
    if (!g) fail(kParameter, "group is NULL");
    if (size) *size = (int32_t)g->ctx.size();
    if (loopback) *loopback = g->loopback ? 1 : 0;
  });
}

int32_t nomad_b200_group_context(nomad_b200_group* g, int32_t rank, nomad_b200_ctx** out) {
  return guard([&] {
    if (!g || !out) fail(kParameter, "NULL argument");
    if (rank < 0 || rank >= (int32_t)g->ctx.size()) fail(kParameter, "rank out of range");
    *out = g->ctx[rank];
  });
}

}  // extern "C"
