timeout 600 python -m pytest tests/test_io_gpu.py tests/test_sgd_gpu.py -x -q --timeout 300 2>&1 | tail -3
timeout 300 python bench.py --steps 8 --warmup 3 > gpurun_out/bench_df.json 2> gpurun_out/bench_df.err; tail -1 gpurun_out/bench_df.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sgd_hogwild -s 2 -c 1 -o gpurun_out/sgd_df python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sgd_df.log 2>&1; tail -2 gpurun_out/ncu_sgd_df.log
