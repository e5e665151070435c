# closing measurement after the lane-pair RED change (run under gpurun from the repo root)
timeout 400 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$? >> gpurun_out/bench_final.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$? >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sgd_hogwild -s 2 -c 1 -o gpurun_out/sgd_pair \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sgd_pair.log 2>&1; echo full=$? >> gpurun_out/ncu_sgd_pair.log
