#!/bin/bash
# Round-1 closing measurement on one B200 (run through gpurun from the repo root).
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/f2_tests.log 2>&1; tail -2 gpurun_out/f2_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo "smoke rc $?"
python bench.py > gpurun_out/f2_bench.json 2> gpurun_out/f2_bench.err; echo "bench rc $?"
python bench.py --impl reference > gpurun_out/f2_ref.json 2> gpurun_out/f2_ref.err; echo "ref rc $?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/f2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/f2_ncu_launch.log 2>&1; echo "launch list rc $?"
ncu --kernel-name regex:k_knn_tc2 -c 1 --set full --import-source on --clock-control none \
    -o gpurun_out/f2_tc2_1m python tools/knn_probe.py 1000000 768 8 bf16 64 \
    > gpurun_out/f2_tc2.log 2>&1; echo "tc2 ncu rc $?"
