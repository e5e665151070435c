// Shard plan (host): shard_clusters' LPT assignment of clusters to logical
// workers (optimizer.hpp:106-144), workers to ranks in contiguous blocks, and
// the static slot layout of the per-epoch means all-gather. Shared by the
// trainer and the C-ABI (so multi-rank host logic is testable without GPUs).
#include <algorithm>
#include <cmath>
#include <numeric>

#include "common.cuh"
#include "plan.cuh"

namespace nb {

std::vector<double> inverse_rank_weights(uint64_t k) {
  std::vector<double> w(k);
  double total = 0.0;
  for (uint64_t t = 1; t <= k; ++t) {
    w[t - 1] = std::exp(1.0 / static_cast<double>(t));
    total += w[t - 1];
  }
  for (double& x : w) x /= total;
  return w;
}

std::vector<double> weight_table(uint64_t k) {
  std::vector<double> wt((k + 1) * k, 0.0);
  for (uint64_t c = 1; c <= k; ++c) {
    auto w = inverse_rank_weights(c);
    std::copy(w.begin(), w.end(), wt.begin() + c * k);
  }
  return wt;
}

ShardPlan make_plan(const std::vector<uint32_t>& sizes, uint32_t W, int world) {
  const uint32_t C = (uint32_t)sizes.size();
  if (W < 1) fail(kParameter, "workers must be >= 1");
  if (C < W)
    fail(kParameter, "clusters must be >= workers (" + std::to_string(C) + " < " +
                         std::to_string(W) + ")");
  if (world < 1 || W % (uint32_t)world != 0)
    fail(kParameter, "workers must be a multiple of world_size");
  ShardPlan P;
  std::vector<uint32_t> order(C);
  std::iota(order.begin(), order.end(), 0u);
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    if (sizes[a] != sizes[b]) return sizes[a] > sizes[b];
    return a < b;
  });
  P.c2w.assign(C, 0);
  P.wclusters.assign(W, {});
  std::vector<uint64_t> load(W, 0);
  for (uint32_t c : order) {
    uint32_t light = 0;
    for (uint32_t w = 1; w < W; ++w)
      if (load[w] < load[light]) light = w;
    P.c2w[c] = light;
    P.wclusters[light].push_back(c);
    load[light] += sizes[c];
  }
  for (auto& v : P.wclusters) std::sort(v.begin(), v.end());
  const uint32_t nwl = W / world;
  std::vector<uint32_t> per_rank(world, 0);
  for (uint32_t r = 0; r < C; ++r) ++per_rank[P.c2w[r] / nwl];
  P.max_slots = *std::max_element(per_rank.begin(), per_rank.end());
  P.slot_cluster.assign((size_t)world * P.max_slots, 0xFFFFFFFFu);
  for (int rk = 0; rk < world; ++rk) {
    uint32_t q = 0;
    for (uint32_t wl = 0; wl < nwl; ++wl)
      for (uint32_t c : P.wclusters[rk * nwl + wl]) P.slot_cluster[(size_t)rk * P.max_slots + q++] = c;
  }
  return P;
}

}  // namespace nb

using namespace nb;

extern "C" int32_t nomad_b200_plan(uint64_t n, uint64_t C, const uint32_t* assignment,
                                   uint64_t workers, int32_t world, uint32_t* cluster_to_worker,
                                   uint32_t* slot_cluster, uint32_t* max_slots) {
  return guard([&] {
    if (!assignment || !cluster_to_worker || !max_slots) fail(kParameter, "NULL argument");
    std::vector<uint32_t> sizes(C, 0);
    for (uint64_t i = 0; i < n; ++i) {
      if (assignment[i] >= C) fail(kParameter, "assignment entry out of range");
      ++sizes[assignment[i]];
    }
    ShardPlan P = make_plan(sizes, (uint32_t)workers, world);
    std::copy(P.c2w.begin(), P.c2w.end(), cluster_to_worker);
    if (slot_cluster) std::copy(P.slot_cluster.begin(), P.slot_cluster.end(), slot_cluster);
    *max_slots = P.max_slots;
  });
}
