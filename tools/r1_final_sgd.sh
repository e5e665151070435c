timeout 300 python bench.py --steps 8 --warmup 3 > gpurun_out/bench_pf.json 2> gpurun_out/bench_pf.err; tail -1 gpurun_out/bench_pf.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_pf.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_pf.log 2>&1; tail -1 gpurun_out/ncu_launch_pf.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sgd_hogwild -s 2 -c 1 -o gpurun_out/sgd_pf python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sgd_pf.log 2>&1; tail -1 gpurun_out/ncu_sgd_pf.log
timeout 1500 python tools/quality_scale.py 1000000 768 64 8 100 8
