#!/bin/bash
# compute-sanitizer passes over the small GPU tests (one B200, gpurun):
# memcheck (out-of-bounds / misaligned device accesses, leaks of device
# errors) and synccheck (barrier misuse) on the SGD (replay dataflow,
# hogwild), group, k-means, kNN and metrics paths. Each pass bounded by timeout.
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL_SGD='test_replay_bit_exact or test_replay_repeated_list_entries or test_replay_ragged or test_divergence or test_hogwild_statistical_parity or test_many_clusters or test_hogwild_ablation'
run() {  # tool, label, pytest args...
  local tool=$1 label=$2; shift 2
  timeout 1500 $CS --tool $tool --target-processes all --error-exitcode 99 --print-limit 20 \
    python -m pytest -q -x -m gpu -p no:cacheprovider "$@" > gpurun_out/san_${tool}_${label}.log 2>&1
  echo "$tool $label rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/san_${tool}_${label}.log | tail -2 | tr '\n' ' ')"
}
run memcheck sgd tests/test_sgd_gpu.py -k "$SEL_SGD"
run memcheck group tests/test_group_gpu.py
run memcheck kmeans tests/test_kmeans_gpu.py
run memcheck knn tests/test_knn_gpu.py -k "not multiblob"
run memcheck metrics tests/test_metrics_gpu.py
run synccheck sgd tests/test_sgd_gpu.py -k "test_replay_bit_exact or test_hogwild_statistical_parity"
run synccheck knn tests/test_knn_gpu.py -k "test_knn_bit_exact"
