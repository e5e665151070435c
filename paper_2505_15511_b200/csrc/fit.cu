// fit() (optimizer.hpp:327-482) composed from the engine's own entry points
// with every intermediate kept on the device: lsh_init -> kmeans_em ->
// build_knn -> (pca_init) -> trainer epochs. The dataset is uploaded once.
#include <algorithm>
#include <cstring>
#include <initializer_list>

#include "index_common.cuh"

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
}  // namespace
}  // namespace nb

using namespace nb;

extern "C" int32_t nomad_b200_fit(nomad_b200_ctx* ctx, const nomad_b200_dataset_view* data,
                                  const nomad_b200_train_config* cfg, const double* init_layout,
                                  double* layout_out, nomad_b200_clusters* clusters_out,
                                  nomad_b200_graph* graph_out, double* epoch_loss_out) {
  return guard([&] {
    if (!ctx || !data || !cfg || !layout_out) fail(kParameter, "NULL argument");
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
    DevData dd;
    dd.bind(data, S);
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
      chk(nomad_b200_kmeans_em_default_tol(ctx, &dv, &cl, cfg->kmeans_max_iters, nullptr,
                                           nullptr));
    DBuf<uint32_t> off(n + 1), nbr(std::max<uint64_t>(n * k, 1));
    DBuf<double> dist(std::max<uint64_t>(n * k, 1));
    nomad_b200_graph g{n, k, off.p, nbr.p, dist.p, NOMAD_B200_DEVICE};
    chk(nomad_b200_build_knn(ctx, &dv, &cl, k, cfg->knn_mode, &g));  // :341

    DBuf<double> init(2 * n);
    if (init_layout) {
      NB_CUDA(cudaMemcpyAsync(init.p, init_layout, n * 16, cudaMemcpyHostToDevice, S));
    } else {
      // :353 — bit-identical PCA where the trajectory is (replay), the
      // precomputed-covariance form in throughput mode
      if (cfg->sgd_mode == NOMAD_B200_SGD_HOGWILD)
        chk(nomad_b200_pca_init_fast(ctx, &dv, cfg->seed, init.p, NOMAD_B200_DEVICE));
      else
        chk(nomad_b200_pca_init(ctx, &dv, cfg->seed, init.p, NOMAD_B200_DEVICE));
    }
    nomad_b200_trainer* tr = nullptr;
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
          const std::string path = std::string(cfg->checkpoint_prefix) + ".epoch" + std::to_string(e) + ".csv";
          rc = nomad_b200_save_layout_csv(path.c_str(), layout_out, n, cfg->checkpoint_ids,
                                          cfg->checkpoint_labels);
        }
      }
    }
    if (rc == 0) rc = nomad_b200_trainer_layout(tr, layout_out, NOMAD_B200_HOST);
    if (rc) msg = nomad_b200_last_error();
    nomad_b200_trainer_destroy(tr);
    if (rc) throw Error(static_cast<Kind>(rc - 1), msg);

    if (clusters_out) {
      const auto kind = clusters_out->location == NOMAD_B200_DEVICE ? cudaMemcpyDeviceToDevice
                                                                    : cudaMemcpyDeviceToHost;
      if (clusters_out->assignment)
        NB_CUDA(cudaMemcpyAsync(clusters_out->assignment, a.p, n * 4, kind, S));
      if (clusters_out->centroids)
        NB_CUDA(cudaMemcpyAsync(clusters_out->centroids, cent.p, C * d * 8, kind, S));
      if (clusters_out->sizes) NB_CUDA(cudaMemcpyAsync(clusters_out->sizes, sizes.p, C * 4, kind, S));
      clusters_out->rows = n;
      clusters_out->n_clusters = C;
      clusters_out->dims = d;
    }
    if (graph_out) {
      const auto kind = graph_out->location == NOMAD_B200_DEVICE ? cudaMemcpyDeviceToDevice
                                                                 : cudaMemcpyDeviceToHost;
      uint32_t edges = 0;
      NB_CUDA(cudaMemcpy(&edges, off.p + n, 4, cudaMemcpyDeviceToHost));
      NB_CUDA(cudaMemcpyAsync(graph_out->offsets, off.p, (n + 1) * 4, kind, S));
      if (edges) {
        NB_CUDA(cudaMemcpyAsync(graph_out->neighbors, nbr.p, (uint64_t)edges * 4, kind, S));
        if (graph_out->distances)
          NB_CUDA(cudaMemcpyAsync(graph_out->distances, dist.p, (uint64_t)edges * 8, kind, S));
      }
      graph_out->rows = n;
      graph_out->k = k;
    }
    NB_CUDA(cudaStreamSynchronize(S));
  });
}
