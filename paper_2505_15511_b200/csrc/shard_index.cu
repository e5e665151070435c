// Row-sharded index build (the 60M-row configuration across
// GPUs): every rank holds only its share of the rows.
//
//   lsh_init + kmeans_em   row-sharded (kmeans.cu with a Comm): integer
//                          counts all-reduced, every ascending-id sum carried
//                          rank to rank -> bit-identical to one GPU;
//   shard_clusters         the LPT plan (optimizer.hpp:106-144) over W
//                          workers, workers in contiguous rank blocks;
//   rows -> owners         one all-to-all: each row goes to the rank that
//                          owns its cluster (ascending point id kept);
//   build_knn              on the owned clusters' rows (clusters are the
//                          graph's components, knn.hpp:62-64), ids mapped
//                          back to global point ids -> the one-GPU lists.
#include <algorithm>
#include <cstring>
#include <exception>
#include <memory>
#include <thread>

#include "index_common.cuh"
#include "plan.cuh"
#include "shard.cuh"

extern "C" int32_t nomad_b200_build_knn(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                        const nomad_b200_clusters* clusters, uint64_t k,
                                        int32_t knn_mode, nomad_b200_graph* out);

namespace nb {

// kmeans.cu: the row-sharded forms of lsh_init / kmeans_em (km.comm set)
void sharded_kmeans(nomad_b200_ctx* ctx, Comm* comm, XPtr x, uint64_t n, uint64_t row0,
                    uint64_t n_total, uint64_t d, uint32_t C, uint64_t seed, uint64_t max_iters,
                    double tol, std::vector<uint32_t>& a_local, std::vector<double>& cent,
                    std::vector<uint32_t>& sizes);

namespace {

__global__ void k_gather_rows_u32(const uint32_t* src, const uint32_t* idx, uint64_t m,
                                  uint32_t words, uint32_t* dst) {
  const uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (e >= m * words) return;
  const uint64_t r = e / words, w = e % words;
  dst[e] = src[(uint64_t)idx[r] * words + w];
}

struct ShardOut {
  std::vector<uint32_t> assign;         // n_total
  std::vector<double> cent;             // C x d
  std::vector<uint32_t> sizes;          // C
  std::vector<uint32_t> gid;            // received rows: global ids (ascending)
  std::vector<uint32_t> off;            // received rows' CSR (local)
  std::vector<uint32_t> nbr;            // neighbour global ids
  std::vector<double> dist;
};

void index_rank(nomad_b200_ctx* ctx, Comm* comm, const nomad_b200_dataset_view* rows,
                uint64_t row0, uint64_t n_total, uint64_t C, uint64_t seed, uint64_t max_iters,
                double tol, uint64_t W, uint64_t k, int32_t knn_mode, ShardOut& out) {
  cudaStream_t S = ctx->stream;
  DevData dd;
  dd.bind(rows, ctx);
  const uint64_t n = dd.n, d = dd.d;
  const int world = comm->world, rank = comm->rank;
  if (W % (uint64_t)world) fail(kParameter, "workers must be a multiple of world_size");
  // every rank's row range (contiguous, rank order)
  std::vector<uint64_t> rr(2 * (size_t)world);
  {
    const uint64_t mine[2] = {row0, n};
    comm->allgather(mine, 16, rr.data());
    uint64_t expect = 0;
    for (int r = 0; r < world; ++r) {
      if (rr[2 * r] != expect) fail(kParameter, "row ranges must tile [0, n_total) in rank order");
      expect += rr[2 * r + 1];
    }
    if (expect != n_total) fail(kParameter, "row ranges do not cover n_total rows");
  }
  // 1. row-sharded LSH + Lloyd (bit-identical to one GPU)
  std::vector<uint32_t> a_local;
  sharded_kmeans(ctx, comm, dd.x, n, row0, n_total, d, (uint32_t)C, seed, max_iters, tol, a_local,
                 out.cent, out.sizes);
  // global assignment (padded all-gather)
  {
    uint64_t mx = 0;
    for (int r = 0; r < world; ++r) mx = std::max(mx, rr[2 * r + 1]);
    std::vector<uint32_t> pad(mx, 0), all(mx * world);
    std::copy(a_local.begin(), a_local.end(), pad.begin());
    comm->allgather(pad.data(), mx * 4, all.data());
    out.assign.resize(n_total);
    for (int r = 0; r < world; ++r)
      std::copy(all.begin() + (size_t)r * mx, all.begin() + (size_t)r * mx + rr[2 * r + 1],
                out.assign.begin() + rr[2 * r]);
  }
  // 2. shard plan: cluster -> worker -> rank
  const ShardPlan P = make_plan(out.sizes, (uint32_t)W, world);
  const uint32_t nwl = (uint32_t)(W / world);
  auto owner = [&](uint32_t c) { return (int)(P.c2w[c] / nwl); };
  // 3. rows to their owners (stable by destination: ascending point id)
  std::vector<uint64_t> cnt(world, 0);
  for (uint64_t i = 0; i < n; ++i) ++cnt[owner(a_local[i])];
  std::vector<uint64_t> first(world + 1, 0);
  for (int p = 0; p < world; ++p) first[p + 1] = first[p] + cnt[p];
  std::vector<uint32_t> order(n), sid(n), slab(n);
  {
    std::vector<uint64_t> f(first.begin(), first.end() - 1);
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t at = f[owner(a_local[i])]++;
      order[at] = (uint32_t)i;
      sid[at] = (uint32_t)(row0 + i);
      slab[at] = a_local[i];
    }
  }
  std::vector<uint64_t> allcnt((size_t)world * world);
  comm->allgather(cnt.data(), (size_t)world * 8, allcnt.data());
  uint64_t m = 0;
  std::vector<uint64_t> from(world + 1, 0);
  for (int p = 0; p < world; ++p) {
    from[p + 1] = from[p] + allcnt[(size_t)p * world + rank];
    m = from[p + 1];
  }
  const uint32_t elem = dd.x.bf ? 2 : 4;
  const uint64_t rb = d * elem;
  if (rb % 4) fail(kParameter, "row-sharded build needs rows of a multiple of 4 bytes");
  DBuf<uint32_t> didx(std::max<uint64_t>(n, 1));
  DBuf<uint8_t> sendb(std::max<uint64_t>(n * rb, 1)), recvb(std::max<uint64_t>(m * rb, 1));
  DBuf<uint32_t> sidd(std::max<uint64_t>(n, 1)), rid(std::max<uint64_t>(m, 1));
  DBuf<uint32_t> slabd(std::max<uint64_t>(n, 1)), rlab(std::max<uint64_t>(m, 1));
  NB_CUDA(cudaMemcpyAsync(didx.p, order.data(), n * 4, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(sidd.p, sid.data(), n * 4, cudaMemcpyHostToDevice, S));
  NB_CUDA(cudaMemcpyAsync(slabd.p, slab.data(), n * 4, cudaMemcpyHostToDevice, S));
  {
    const uint32_t words = (uint32_t)(rb / 4);
    const uint64_t e = n * words;
    k_gather_rows_u32<<<(unsigned)((e + 255) / 256), 256, 0, S>>>(
        static_cast<const uint32_t*>(dd.x.p), didx.p, n, words, reinterpret_cast<uint32_t*>(sendb.p));
    note_launch(ctx, "k_gather_rows_u32");
  }
  NB_CUDA(cudaStreamSynchronize(S));
  auto scaled = [&](const std::vector<uint64_t>& v, uint64_t s) {
    std::vector<uint64_t> o(v.size());
    for (size_t i = 0; i < v.size(); ++i) o[i] = v[i] * s;
    return o;
  };
  comm->alltoallv(sendb.p, scaled(first, rb).data(), recvb.p, scaled(from, rb).data());
  comm->alltoallv(sidd.p, scaled(first, 4).data(), rid.p, scaled(from, 4).data());
  comm->alltoallv(slabd.p, scaled(first, 4).data(), rlab.p, scaled(from, 4).data());
  sendb.release();
  // 4. kNN lists of the owned clusters, on the received rows
  out.gid.resize(m);
  if (m) NB_CUDA(cudaMemcpy(out.gid.data(), rid.p, m * 4, cudaMemcpyDeviceToHost));
  out.off.assign(m + 1, 0);
  out.nbr.clear();
  out.dist.clear();
  if (m) {
    nomad_b200_dataset_view lv{m, d, reinterpret_cast<const float*>(recvb.p), NOMAD_B200_DEVICE,
                               dd.x.bf ? NOMAD_B200_BF16 : NOMAD_B200_F32};
    nomad_b200_clusters lc{m, C, d, rlab.p, nullptr, nullptr, NOMAD_B200_DEVICE};
    std::vector<uint32_t> lnb(m * k);
    out.dist.resize(m * k);
    nomad_b200_graph g{m, k, out.off.data(), lnb.data(), out.dist.data(), NOMAD_B200_HOST};
    const int32_t rc = nomad_b200_build_knn(ctx, &lv, &lc, k, knn_mode, &g);
    if (rc) throw Error(static_cast<Kind>(rc - 1), nomad_b200_last_error());
    const uint64_t e = out.off[m];
    out.nbr.resize(e);
    out.dist.resize(e);
    for (uint64_t t = 0; t < e; ++t) out.nbr[t] = out.gid[lnb[t]];
  }
}

// The rank's lists into a global CSR over n_total rows (other rows empty),
// or merged into `graph` (rows not listed stay as they are: zero counts).
void to_global(const ShardOut& o, uint64_t n_total, std::vector<uint32_t>& cnt) {
  for (size_t i = 0; i < o.gid.size(); ++i) cnt[o.gid[i]] = o.off[i + 1] - o.off[i];
}

void write_outputs(const std::vector<const ShardOut*>& parts, uint64_t n_total, uint64_t C,
                   uint64_t d, nomad_b200_clusters* cl, nomad_b200_graph* g) {
  const ShardOut& o0 = *parts[0];
  if (cl) {
    if (cl->location == NOMAD_B200_DEVICE) fail(kParameter, "sharded outputs are host buffers");
    if (cl->assignment) std::memcpy(cl->assignment, o0.assign.data(), n_total * 4);
    if (cl->centroids) std::memcpy(cl->centroids, o0.cent.data(), C * d * 8);
    if (cl->sizes) std::memcpy(cl->sizes, o0.sizes.data(), C * 4);
    cl->rows = n_total;
    cl->n_clusters = C;
    cl->dims = d;
  }
  if (g) {
    if (g->location == NOMAD_B200_DEVICE) fail(kParameter, "sharded outputs are host buffers");
    std::vector<uint32_t> cnt(n_total, 0);
    for (auto* p : parts) to_global(*p, n_total, cnt);
    g->offsets[0] = 0;
    for (uint64_t i = 0; i < n_total; ++i) g->offsets[i + 1] = g->offsets[i] + cnt[i];
    for (auto* p : parts)
      for (size_t i = 0; i < p->gid.size(); ++i) {
        const uint32_t b = p->off[i], e = p->off[i + 1], at = g->offsets[p->gid[i]];
        std::copy(p->nbr.begin() + b, p->nbr.begin() + e, g->neighbors + at);
        if (g->distances)
          std::copy(p->dist.begin() + b, p->dist.begin() + e, g->distances + at);
      }
    g->rows = n_total;
  }
}

}  // namespace
}  // namespace nb

using namespace nb;

extern "C" {

int32_t nomad_b200_index_sharded(nomad_b200_ctx* ctx, int32_t rank, int32_t world,
                                 const void* nccl_id, const nomad_b200_dataset_view* rows,
                                 uint64_t row0, uint64_t n_total, uint64_t n_clusters,
                                 uint64_t seed, uint64_t kmeans_max_iters, double kmeans_tol,
                                 uint64_t workers, uint64_t k, int32_t knn_mode,
                                 nomad_b200_clusters* clusters_out, nomad_b200_graph* graph_out) {
  return guard([&] {
    if (!ctx || !rows) fail(kParameter, "NULL argument");
    if (world < 1 || rank < 0 || rank >= world) fail(kParameter, "bad rank / world_size");
    bind_device(ctx);
    std::unique_ptr<Comm> comm(make_nccl_comm(rank, world, nccl_id, ctx->stream));
    ShardOut o;
    index_rank(ctx, comm.get(), rows, row0, n_total, n_clusters, seed, kmeans_max_iters,
               kmeans_tol, workers, k, knn_mode, o);
    write_outputs({&o}, n_total, n_clusters, rows->dims, clusters_out, graph_out);
  });
}

int32_t nomad_b200_group_index_sharded(nomad_b200_group* grp, const nomad_b200_dataset_view* rows,
                                       const uint64_t* row0, uint64_t n_total,
                                       uint64_t n_clusters, uint64_t seed,
                                       uint64_t kmeans_max_iters, double kmeans_tol,
                                       uint64_t workers, uint64_t k, int32_t knn_mode,
                                       nomad_b200_clusters* clusters_out,
                                       nomad_b200_graph* graph_out) {
  return guard([&] {
    if (!grp || !rows || !row0) fail(kParameter, "NULL argument");
    const int G = (int)grp->ctx.size();
    GroupRendezvous* rz = make_rendezvous(G);
    std::vector<ShardOut> outs(G);
    std::vector<std::exception_ptr> errs(G);
    std::vector<std::thread> th;
    for (int r = 0; r < G; ++r)
      th.emplace_back([&, r] {
        nomad_b200_ctx* c = grp->ctx[r];
        cudaStream_t shared = c->stream;
        cudaStream_t own = nullptr;
        try {
          bind_device(c);
          // a private stream per rank thread (loopback ranks share one)
          NB_CUDA(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
          c->stream = own;
          std::unique_ptr<Comm> comm(make_group_comm(rz, r, own, c->device));
          index_rank(c, comm.get(), rows + r, row0[r], n_total, n_clusters, seed,
                     kmeans_max_iters, kmeans_tol, workers, k, knn_mode, outs[r]);
        } catch (...) {
          errs[r] = std::current_exception();
          rendezvous_abort(rz);
        }
        if (own) {
          cudaStreamSynchronize(own);
          cudaStreamDestroy(own);
        }
        c->stream = shared;
      });
    for (auto& t : th) t.join();
    free_rendezvous(rz);
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    std::vector<const ShardOut*> parts;
    for (auto& o : outs) parts.push_back(&o);
    write_outputs(parts, n_total, n_clusters, rows[0].dims, clusters_out, graph_out);
  });
}

}  // extern "C"
