// Row-sharded execution of the index build across the ranks of a multi-GPU
// run: rank r holds the rows [row0, row0 + n) of an n_total-row
// dataset. Integer quantities (sizes, changes, bucket counts) are all-reduced;
// every floating-point sum the reference accumulates in ascending point id
// (kmeans.hpp:90-104 centroids, :176-181 data mean, :218-226 bucket means,
// :148-154 quantization error, :157-161 tolerance) is carried rank to rank in
// rank order, so each rank continues the previous rank's running sums and the
// results are bit-identical to one GPU's.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <vector>

namespace nb {

struct Comm {
  int rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  virtual ~Comm() = default;
  // in-place sum over ranks of a host u64 vector
  virtual void allreduce_u64(uint64_t* v, size_t n) = 0;
  // the carry chain: rank 0 starts from zeros, every other rank from the
  // previous rank's result; step() continues the sums in `dev` (n doubles,
  // this rank's device) on this rank's stream; on return every rank holds the
  // last rank's result
  virtual void chain(double* dev, size_t n, const std::function<void()>& step) = 0;
  // host bytes of every rank, rank-major into `all` (world * bytes)
  virtual void allgather(const void* mine, size_t bytes, void* all) = 0;
  // device all-to-all: this rank sends send[soff[p], soff[p+1]) bytes to rank
  // p and receives rank p's slice into recv[roff[p], roff[p+1])
  virtual void alltoallv(const void* send, const uint64_t* soff, void* recv,
                         const uint64_t* roff) = 0;
};

// One process per GPU: NCCL (send/recv for the chain, all-reduce, all-gather,
// grouped send/recv for the all-to-all).
Comm* make_nccl_comm(int rank, int world, const void* nccl_id, cudaStream_t stream);

// Every rank of a group in its own host thread (one process): a shared
// rendezvous, host staging for the chain, peer copies for the all-to-all.
struct GroupRendezvous;
GroupRendezvous* make_rendezvous(int world);
void free_rendezvous(GroupRendezvous* g);
// a rank failed: wake every waiting rank (their waits throw)
void rendezvous_abort(GroupRendezvous* g);
Comm* make_group_comm(GroupRendezvous* g, int rank, cudaStream_t stream, int device);

}  // namespace nb
