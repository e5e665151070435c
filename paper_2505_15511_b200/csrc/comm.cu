// Rank-to-rank primitives of the row-sharded index build (shard.cuh): NCCL
// between processes, or a host rendezvous between the threads that drive the
// ranks of a group in one process.
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "shard.cuh"

namespace nb {

#define NB_NCCL2(call)                                                              \
  do {                                                                              \
    ncclResult_t r_ = (call);                                                       \
    if (r_ != ncclSuccess) fail(kInternal, std::string("NCCL error: ") + ncclGetErrorString(r_)); \
  } while (0)

namespace {

struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) ncclCommDestroy(c);
  }
  void allreduce_u64(uint64_t* v, size_t n) override {
    if (!n || world == 1) return;
    DBuf<uint64_t> d(n);
    NB_CUDA(cudaMemcpyAsync(d.p, v, n * 8, cudaMemcpyHostToDevice, stream));
    NB_NCCL2(ncclAllReduce(d.p, d.p, n, ncclUint64, ncclSum, c, stream));
    NB_CUDA(cudaMemcpyAsync(v, d.p, n * 8, cudaMemcpyDeviceToHost, stream));
    NB_CUDA(cudaStreamSynchronize(stream));
  }
  void chain(double* dev, size_t n, const std::function<void()>& step) override {
    if (rank == 0) NB_CUDA(cudaMemsetAsync(dev, 0, n * 8, stream));
    else NB_NCCL2(ncclRecv(dev, n, ncclDouble, rank - 1, c, stream));
    step();
    if (world > 1) {
      if (rank + 1 < world) NB_NCCL2(ncclSend(dev, n, ncclDouble, rank + 1, c, stream));
      NB_NCCL2(ncclBroadcast(dev, dev, n, ncclDouble, world - 1, c, stream));
    }
    NB_CUDA(cudaStreamSynchronize(stream));
  }
  void allgather(const void* mine, size_t bytes, void* all) override {
    if (world == 1) {
      std::memcpy(all, mine, bytes);
      return;
    }
    DBuf<uint8_t> a(std::max<size_t>(bytes, 1)), b(std::max<size_t>(bytes * world, 1));
    NB_CUDA(cudaMemcpyAsync(a.p, mine, bytes, cudaMemcpyHostToDevice, stream));
    NB_NCCL2(ncclAllGather(a.p, b.p, bytes, ncclChar, c, stream));
    NB_CUDA(cudaMemcpyAsync(all, b.p, bytes * world, cudaMemcpyDeviceToHost, stream));
    NB_CUDA(cudaStreamSynchronize(stream));
  }
  void alltoallv(const void* send, const uint64_t* soff, void* recv,
                 const uint64_t* roff) override {
    if (world == 1) {
      if (soff[1] > soff[0])
        NB_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + roff[0],
                                static_cast<const char*>(send) + soff[0], soff[1] - soff[0],
                                cudaMemcpyDeviceToDevice, stream));
      NB_CUDA(cudaStreamSynchronize(stream));
      return;
    }
    NB_NCCL2(ncclGroupStart());
    for (int p = 0; p < world; ++p) {
      const uint64_t sb = soff[p + 1] - soff[p], rb = roff[p + 1] - roff[p];
      if (sb) NB_NCCL2(ncclSend(static_cast<const char*>(send) + soff[p], sb, ncclChar, p, c, stream));
      if (rb) NB_NCCL2(ncclRecv(static_cast<char*>(recv) + roff[p], rb, ncclChar, p, c, stream));
    }
    NB_NCCL2(ncclGroupEnd());
    NB_CUDA(cudaStreamSynchronize(stream));
  }
};

}  // namespace

Comm* make_nccl_comm(int rank, int world, const void* nccl_id, cudaStream_t stream) {
  auto* m = new NcclComm();
  m->rank = rank;
  m->world = world;
  m->stream = stream;
  if (world > 1) {
    if (!nccl_id) fail(kParameter, "nccl_id required when world_size > 1");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof id);
    ncclResult_t r = ncclCommInitRank(&m->c, world, id, rank);
    if (r != ncclSuccess) {
      delete m;
      fail(kInternal, std::string("NCCL error: ") + ncclGetErrorString(r));
    }
  }
  return m;
}

// ------------------------------------------------------------- group form
struct GroupRendezvous {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  uint64_t gen = 0;
  int arrived = 0, turn = 0;
  bool aborted = false;  // a rank failed: every wait throws instead of hanging
  std::vector<double> stage;
  std::vector<const void*> ptrs;
  std::vector<const uint64_t*> offs;
  std::vector<int> devs;
  explicit GroupRendezvous(int w) : world(w), ptrs(w), offs(w), devs(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) fail(kInternal, "a peer rank of the group failed");
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || aborted; });
      if (aborted) fail(kInternal, "a peer rank of the group failed");
    }
  }
};

void rendezvous_abort(GroupRendezvous* g) {
  std::lock_guard<std::mutex> lk(g->mu);
  g->aborted = true;
  g->cv.notify_all();
}

GroupRendezvous* make_rendezvous(int world) { return new GroupRendezvous(world); }
void free_rendezvous(GroupRendezvous* g) { delete g; }

namespace {

struct GroupComm : Comm {
  GroupRendezvous* g = nullptr;
  int device = 0;
  void allreduce_u64(uint64_t* v, size_t n) override {
    g->ptrs[rank] = v;
    g->barrier();
    std::vector<uint64_t> acc(n, 0);
    for (int r = 0; r < world; ++r) {
      const uint64_t* o = static_cast<const uint64_t*>(g->ptrs[r]);
      for (size_t i = 0; i < n; ++i) acc[i] += o[i];
    }
    g->barrier();
    std::memcpy(v, acc.data(), n * 8);
  }
  void chain(double* dev, size_t n, const std::function<void()>& step) override {
    {
      std::unique_lock<std::mutex> lk(g->mu);
      g->cv.wait(lk, [&] { return g->turn == rank || g->aborted; });
      if (g->aborted) fail(kInternal, "a peer rank of the group failed");
    }
    if (rank == 0) NB_CUDA(cudaMemsetAsync(dev, 0, n * 8, stream));
    else NB_CUDA(cudaMemcpyAsync(dev, g->stage.data(), n * 8, cudaMemcpyHostToDevice, stream));
    step();
    g->stage.resize(n);
    NB_CUDA(cudaMemcpyAsync(g->stage.data(), dev, n * 8, cudaMemcpyDeviceToHost, stream));
    NB_CUDA(cudaStreamSynchronize(stream));
    {
      std::lock_guard<std::mutex> lk(g->mu);
      ++g->turn;
      g->cv.notify_all();
    }
    g->barrier();  // the last rank's result is staged
    if (rank + 1 < world)
      NB_CUDA(cudaMemcpyAsync(dev, g->stage.data(), n * 8, cudaMemcpyHostToDevice, stream));
    NB_CUDA(cudaStreamSynchronize(stream));
    if (rank == 0) {
      std::lock_guard<std::mutex> lk(g->mu);
      g->turn = 0;
    }
    g->barrier();  // staging free, turn reset
  }
  void allgather(const void* mine, size_t bytes, void* all) override {
    g->ptrs[rank] = mine;
    g->barrier();
    for (int r = 0; r < world; ++r)
      std::memcpy(static_cast<char*>(all) + (size_t)r * bytes, g->ptrs[r], bytes);
    g->barrier();
  }
  void alltoallv(const void* send, const uint64_t* soff, void* recv,
                 const uint64_t* roff) override {
    g->ptrs[rank] = send;
    g->offs[rank] = soff;
    g->devs[rank] = device;
    g->barrier();
    for (int p = 0; p < world; ++p) {
      const uint64_t b = g->offs[p][rank + 1] - g->offs[p][rank];
      if (b)
        NB_CUDA(cudaMemcpyPeerAsync(static_cast<char*>(recv) + roff[p], device,
                                    static_cast<const char*>(g->ptrs[p]) + g->offs[p][rank],
                                    g->devs[p], b, stream));
    }
    NB_CUDA(cudaStreamSynchronize(stream));
    g->barrier();
  }
};

}  // namespace

Comm* make_group_comm(GroupRendezvous* g, int rank, cudaStream_t stream, int device) {
  auto* m = new GroupComm();
  m->g = g;
  m->rank = rank;
  m->world = g->world;
  m->stream = stream;
  m->device = device;
  return m;
}

}  // namespace nb
