// fit() (optimizer.hpp:327-482) composed from the engine's own entry points
// with every intermediate kept on the device: lsh_init -> kmeans_em ->
// build_knn -> (pca_init) -> trainer epochs (one context, or every rank of a
// group). The dataset is uploaded once; the FitReport (optimizer.hpp:312-321)
// is filled from the engine's outputs (affinity weights and eligible heads by
// a device pass over the graph, the plan and final means from the trainer).
#include <algorithm>
#include <cstring>
#include <initializer_list>

#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "index_common.cuh"
#include "plan.cuh"

extern "C" {
int32_t nomad_b200_pca_init(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                            uint64_t seed, double* layout_out, int32_t location);
int32_t nomad_b200_pca_init_fast(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                 uint64_t seed, double* layout_out, int32_t location);
}

namespace nb {
namespace {
void chk(int32_t rc) {
  if (rc != 0) throw Error(static_cast<Kind>(rc - 1), nomad_b200_last_error());
}

// affinity.hpp:65-84 build_affinity on the device: every edge of a list of c
// neighbours gets row c of the inverse-rank table; eligible = c > 0.
__global__ void k_affinity(const uint32_t* off, uint64_t n, uint32_t k, const double* wtab,
                           double* w, uint8_t* elig) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t b = off[i], c = off[i + 1] - b;
  for (uint32_t t = 0; t < c; ++t) w[b + t] = wtab[(size_t)c * k + t];
  elig[i] = c > 0;
}
}  // namespace
}  // namespace nb

using namespace nb;

static void fit_impl(nomad_b200_ctx* ctx, nomad_b200_group* grp, const nomad_b200_dataset_view* data,
                     const nomad_b200_train_config* cfg, const double* init_layout,
                     double* layout_out, nomad_b200_clusters* clusters_out,
                     nomad_b200_graph* graph_out, double* epoch_loss_out,
                     nomad_b200_fit_report* rep) {
  if (!data || !cfg || !layout_out) fail(kParameter, "NULL argument");
  if (!ctx) {
    if (!grp || grp->ctx.empty()) fail(kParameter, "NULL argument");
    ctx = grp->ctx[0];  // the index is built on rank 0's device
  }
  bind_device(ctx);
  cudaStream_t S = ctx->stream;
  // optimizer.hpp:63-71, :329-334
  if (cfg->workers < 1) fail(kParameter, "workers must be >= 1");
  if (cfg->k < 1) fail(kParameter, "k must be >= 1");
  if (cfg->negatives < 1) fail(kParameter, "negatives must be >= 1");
  if (cfg->local_draws < 1) fail(kParameter, "local draws must be >= 1");
  if (cfg->batch_size < 1) fail(kParameter, "batch size must be >= 1");
  if (cfg->n_clusters != 0 && cfg->n_clusters < cfg->workers)
    fail(kParameter, "clusters must be >= workers");
  if (grp && cfg->workers % grp->ctx.size() != 0)
    fail(kParameter, "workers must be a multiple of world_size");
  DevData dd;
  dd.bind(data, ctx);
  const uint64_t n = dd.n, d = dd.d, k = cfg->k;
  uint64_t C = cfg->n_clusters;
  if (C != 0) {
    C = std::min<uint64_t>(C, n);
  } else {
    const uint64_t want = (n + 4095) / 4096;
    C = std::min<uint64_t>(n, std::max<uint64_t>(std::max<uint64_t>(want, cfg->workers), 2));
  }
  if (C < cfg->workers) fail(kParameter, "clusters must be >= workers");
  nomad_b200_dataset_view dv{n, d, static_cast<const float*>(dd.x.p), NOMAD_B200_DEVICE,
                             dd.x.bf ? NOMAD_B200_BF16 : NOMAD_B200_F32};

  DBuf<uint32_t> a(n), sizes(C);
  DBuf<double> cent(C * d);
  nomad_b200_clusters cl{n, C, d, a.p, cent.p, sizes.p, NOMAD_B200_DEVICE};
  chk(nomad_b200_lsh_init(ctx, &dv, C, cfg->seed, &cl));  // optimizer.hpp:336
  if (cfg->kmeans_tol >= 0.0)                             // :337-339
    chk(nomad_b200_kmeans_em(ctx, &dv, &cl, cfg->kmeans_max_iters, cfg->kmeans_tol, nullptr,
                             nullptr));
  else
    chk(nomad_b200_kmeans_em_default_tol(ctx, &dv, &cl, cfg->kmeans_max_iters, nullptr, nullptr));
  DBuf<uint32_t> off(n + 1), nbr(std::max<uint64_t>(n * k, 1));
  DBuf<double> dist(std::max<uint64_t>(n * k, 1));
  nomad_b200_graph g{n, k, off.p, nbr.p, dist.p, NOMAD_B200_DEVICE};
  chk(nomad_b200_build_knn(ctx, &dv, &cl, k, cfg->knn_mode, &g));  // :341

  DBuf<double> init(2 * n);
  if (init_layout) {
    NB_CUDA(cudaMemcpyAsync(init.p, init_layout, n * 16, cudaMemcpyDefault, S));
  } else {
    // :353 — bit-identical PCA where the trajectory is (replay), the
    // precomputed-covariance form in throughput mode
    if (cfg->sgd_mode == NOMAD_B200_SGD_HOGWILD)
      chk(nomad_b200_pca_init_fast(ctx, &dv, cfg->seed, init.p, NOMAD_B200_DEVICE));
    else
      chk(nomad_b200_pca_init(ctx, &dv, cfg->seed, init.p, NOMAD_B200_DEVICE));
  }
  if (rep && rep->pca)
    NB_CUDA(cudaMemcpyAsync(rep->pca, init.p, n * 16, cudaMemcpyDeviceToHost, S));
  NB_CUDA(cudaStreamSynchronize(S));
  nomad_b200_trainer* tr = nullptr;
  if (grp)
    chk(nomad_b200_group_trainer_create(grp, &g, &cl, init.p, NOMAD_B200_DEVICE, cfg, &tr));
  else
    chk(nomad_b200_trainer_create(ctx, &g, &cl, init.p, NOMAD_B200_DEVICE, cfg, 0, 1, nullptr,
                                  &tr));
  int32_t rc = 0;
  // epochs in segments ending at the checkpoint epochs (optimizer.hpp:463-469)
  const bool ckpt = cfg->checkpoint_every > 0 && cfg->checkpoint_prefix && *cfg->checkpoint_prefix;
  std::string msg;
  for (uint64_t e = 0; rc == 0 && e < cfg->epochs;) {
    const uint64_t seg = ckpt ? std::min(cfg->checkpoint_every - e % cfg->checkpoint_every,
                                         cfg->epochs - e)
                              : cfg->epochs - e;
    rc = nomad_b200_trainer_run(tr, seg, epoch_loss_out ? epoch_loss_out + e : nullptr);
    e += seg;
    if (rc == 0 && ckpt && e % cfg->checkpoint_every == 0) {
      rc = nomad_b200_trainer_layout(tr, layout_out, NOMAD_B200_HOST);
      if (rc == 0) {
        const std::string path =
            std::string(cfg->checkpoint_prefix) + ".epoch" + std::to_string(e) + ".csv";
        rc = nomad_b200_save_layout_csv(path.c_str(), layout_out, n, cfg->checkpoint_ids,
                                        cfg->checkpoint_labels);
      }
    }
  }
  if (rc == 0) rc = nomad_b200_trainer_layout(tr, layout_out, NOMAD_B200_HOST);
  if (rc == 0 && rep) {
    if (rep->final_means) rc = nomad_b200_trainer_means(tr, rep->final_means, nullptr);
    if (rc == 0)
      rc = nomad_b200_trainer_comm(tr, &rep->comm_epochs, &rep->comm_messages,
                                   &rep->comm_payload_doubles, &rep->comm_payload_counts);
  }
  if (rc) msg = nomad_b200_last_error();
  nomad_b200_trainer_destroy(tr);
  if (rc) throw Error(static_cast<Kind>(rc - 1), msg);
  bind_device(ctx);

  if (clusters_out) {
    const auto kind = clusters_out->location == NOMAD_B200_DEVICE ? cudaMemcpyDeviceToDevice
                                                                  : cudaMemcpyDeviceToHost;
    if (clusters_out->assignment)
      copy_out(ctx, clusters_out->assignment, a.p, n * 4, clusters_out->location == NOMAD_B200_DEVICE);
    if (clusters_out->centroids)
      NB_CUDA(cudaMemcpyAsync(clusters_out->centroids, cent.p, C * d * 8, kind, S));
    if (clusters_out->sizes) NB_CUDA(cudaMemcpyAsync(clusters_out->sizes, sizes.p, C * 4, kind, S));
    clusters_out->rows = n;
    clusters_out->n_clusters = C;
    clusters_out->dims = d;
  }
  uint32_t edges = 0;
  NB_CUDA(cudaMemcpy(&edges, off.p + n, 4, cudaMemcpyDeviceToHost));
  if (graph_out) {
    const bool dev = graph_out->location == NOMAD_B200_DEVICE;
    copy_out(ctx, graph_out->offsets, off.p, (n + 1) * 4, dev);
    if (edges) {
      copy_out(ctx, graph_out->neighbors, nbr.p, (uint64_t)edges * 4, dev);
      if (graph_out->distances)
        copy_out(ctx, graph_out->distances, dist.p, (uint64_t)edges * 8, dev);
    }
    graph_out->rows = n;
    graph_out->k = k;
  }
  if (rep) {
    rep->n_clusters = C;
    // build_affinity (affinity.hpp:65-84) from the device graph
    if (rep->affinity_weights || rep->eligible_heads) {
      const std::vector<double> wt = weight_table(k);
      DBuf<double> wtab(wt.size()), w(std::max<uint32_t>(edges, 1));
      DBuf<uint8_t> flag(n);
      NB_CUDA(cudaMemcpyAsync(wtab.p, wt.data(), wt.size() * 8, cudaMemcpyHostToDevice, S));
      k_affinity<<<(unsigned)((n + 255) / 256), 256, 0, S>>>(off.p, n, (uint32_t)k, wtab.p, w.p,
                                                              flag.p);
      note_launch(ctx, "k_affinity");
      if (rep->affinity_weights && edges)
        NB_CUDA(cudaMemcpyAsync(rep->affinity_weights, w.p, (uint64_t)edges * 8,
                                cudaMemcpyDeviceToHost, S));
      // eligible heads: the ascending ids of rows with a list (stable compaction)
      DBuf<uint32_t> ids(n);
      DBuf<unsigned long long> cnt(1);
      thrust::counting_iterator<uint32_t> it(0);
      size_t tmp = 0;
      NB_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp, it, flag.p, ids.p, cnt.p, (int64_t)n, S));
      DBuf<uint8_t> tb(std::max<size_t>(tmp, 1));
      NB_CUDA(cub::DeviceSelect::Flagged(tb.p, tmp, it, flag.p, ids.p, cnt.p, (int64_t)n, S));
      unsigned long long ne = 0;
      NB_CUDA(cudaMemcpyAsync(&ne, cnt.p, 8, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
      rep->n_eligible = ne;
      if (rep->eligible_heads && ne)
        NB_CUDA(cudaMemcpyAsync(rep->eligible_heads, ids.p, ne * 4, cudaMemcpyDeviceToHost, S));
    }
    if (rep->cluster_to_worker) {  // shard_clusters (optimizer.hpp:106-144), the trainer's plan
      std::vector<uint32_t> sz(C);
      NB_CUDA(cudaMemcpyAsync(sz.data(), sizes.p, C * 4, cudaMemcpyDeviceToHost, S));
      NB_CUDA(cudaStreamSynchronize(S));
      const ShardPlan P = make_plan(sz, (uint32_t)cfg->workers, 1);
      std::copy(P.c2w.begin(), P.c2w.end(), rep->cluster_to_worker);
    }
  }
  NB_CUDA(cudaStreamSynchronize(S));
}

extern "C" int32_t nomad_b200_fit(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                  const nomad_b200_train_config* cfg, const double* init_layout,
                                  double* layout_out, nomad_b200_clusters* clusters_out,
                                  nomad_b200_graph* graph_out, double* epoch_loss_out) {
  return guard([&] {
    if (!ctx) fail(kParameter, "NULL argument");
    fit_impl(ctx, nullptr, data, cfg, init_layout, layout_out, clusters_out, graph_out,
             epoch_loss_out, nullptr);
  });
}

extern "C" int32_t nomad_b200_fit_ex(nomad_b200_ctx* ctx, nomad_b200_group* group,
                                     const nomad_b200_dataset_view* data,
                                     const nomad_b200_train_config* cfg,
                                     const double* init_layout, double* layout_out,
                                     nomad_b200_fit_report* rep) {
  return guard([&] {
    if ((ctx == nullptr) == (group == nullptr)) fail(kParameter, "exactly one of ctx / group");
    fit_impl(ctx, group, data, cfg, init_layout, layout_out, rep ? rep->clusters : nullptr,
             rep ? rep->graph : nullptr, rep ? rep->epoch_mean_loss : nullptr, rep);
  });
}
