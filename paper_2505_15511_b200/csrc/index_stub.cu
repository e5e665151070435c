// Placeholder entry points for the index build / fit until their kernels land.
#include "common.cuh"
using namespace nb;
extern "C" {
int32_t nomad_b200_default_kmeans_tol(nomad_b200_ctx*, const nomad_b200_dataset_view*, double*) {
  return guard([&] { fail(kInternal, "default_kmeans_tol: not built yet"); });
}
int32_t nomad_b200_lsh_init(nomad_b200_ctx*, const nomad_b200_dataset_view*, uint64_t, uint64_t,
                            nomad_b200_clusters*) {
  return guard([&] { fail(kInternal, "lsh_init: not built yet"); });
}
int32_t nomad_b200_kmeans_em(nomad_b200_ctx*, const nomad_b200_dataset_view*, nomad_b200_clusters*,
                             uint64_t, double, double*, uint64_t*) {
  return guard([&] { fail(kInternal, "kmeans_em: not built yet"); });
}
int32_t nomad_b200_build_knn(nomad_b200_ctx*, const nomad_b200_dataset_view*,
                             const nomad_b200_clusters*, uint64_t, int32_t, nomad_b200_graph*) {
  return guard([&] { fail(kInternal, "build_knn: not built yet"); });
}
int32_t nomad_b200_fit(nomad_b200_ctx*, const nomad_b200_dataset_view*,
                       const nomad_b200_train_config*, const double*, double*,
                       nomad_b200_clusters*, nomad_b200_graph*, double*) {
  return guard([&] { fail(kInternal, "fit: not built yet"); });
}
}
