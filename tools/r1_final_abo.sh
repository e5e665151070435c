# round-1 closing measurement (lane-pair RED.F64 + ABO template), run under gpurun from the repo root
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke=$? >> gpurun_out/smoke_final.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_final.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests_final.log
timeout 400 python bench.py > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err; echo bench=$? >> gpurun_out/bench_final3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches3.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch3.log 2>&1; echo launches=$? >> gpurun_out/ncu_launch3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sgd_hogwild -s 2 -c 1 -o gpurun_out/sgd_abo \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_sgd_abo.log 2>&1; echo full=$? >> gpurun_out/ncu_sgd_abo.log
