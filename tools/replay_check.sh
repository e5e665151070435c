timeout 400 python -m pytest tests/test_sgd_gpu.py tests/test_group_gpu.py tests/test_shard_gpu.py tests/test_fit_gpu.py -q -x -m gpu 2>&1 | tail -2
NOMAD_B200_LIB=$PWD/paper_2505_15511_b200/libnomad_b200_trace.so timeout 300 python tools/replay_chain.py 400000 8 1 2>&1 | grep dftrace | tail -2
timeout 300 python tools/replay_chain.py 400000 8 2
for a in "1000000 8 8 3 synthetic" "1000000 8 8 3 knn" "10000000 64 8 3 synthetic" "10000000 64 8 3 knn"; do timeout 400 python tools/replay_probe.py $a 2>&1 | tail -1; done
