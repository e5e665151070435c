// Placeholder entry points for the index build / fit until their kernels land.
#include "common.cuh"
using namespace nb;
extern "C" {
int32_t nomad_b200_fit(nomad_b200_ctx*, const nomad_b200_dataset_view*,
                       const nomad_b200_train_config*, const double*, double*,
                       nomad_b200_clusters*, nomad_b200_graph*, double*) {
  return guard([&] { fail(kInternal, "fit: not built yet"); });
}
}
