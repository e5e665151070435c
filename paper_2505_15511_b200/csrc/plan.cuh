#pragma once
#include <stdint.h>

#include <vector>

namespace nb {

struct ShardPlan {
  std::vector<uint32_t> c2w;                     // cluster -> worker
  std::vector<std::vector<uint32_t>> wclusters;  // worker -> clusters (ascending)
  std::vector<uint32_t> slot_cluster;            // [world * max_slots] cluster per slot
  uint32_t max_slots = 0;
};

ShardPlan make_plan(const std::vector<uint32_t>& sizes, uint32_t W, int world);

// affinity.hpp:32-42 inverse-rank weights (host libm exp, as the reference).
std::vector<double> inverse_rank_weights(uint64_t k);
// (k + 1) x k table: row c = the weights of a list of c neighbours.
std::vector<double> weight_table(uint64_t k);

}  // namespace nb
