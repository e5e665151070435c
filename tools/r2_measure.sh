#!/bin/bash
# Round-2 measurement run on one B200 (gpurun): tests, smoke, bench, launch list,
# ncu captures of the throughput SGD and the replay dataflow kernel, replay probes.
set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu --timeout 400 2>&1 | tail -6 > gpurun_out/r2_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --replay-epochs 1 > gpurun_out/r2_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sgd_hogwild -s 3 -c 1 \
  -o gpurun_out/r2_sgd python bench.py --steps 1 --warmup 3 --no-cpu-baseline --replay-epochs 0 \
  > gpurun_out/r2_sgd_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sgd_dataflow -c 1 \
  -o gpurun_out/r2_dataflow python tools/replay_probe.py 1000000 8 8 1 knn > gpurun_out/r2_dataflow_ncu.log 2>&1
for a in "1000000 8 8 3 synthetic" "1000000 8 8 3 knn" "10000000 64 8 3 synthetic" "10000000 64 8 3 knn"; do
  timeout 400 python tools/replay_probe.py $a
done > gpurun_out/r2_replay.txt 2>&1
cat gpurun_out/r2_gpu_tests.txt gpurun_out/r2_smoke.txt; tail -c 600 gpurun_out/r2_bench.json; cat gpurun_out/r2_replay.txt
