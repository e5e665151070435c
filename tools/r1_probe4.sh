timeout 300 python tools/knn_probe.py 1000000 768 8 bf16 64
timeout 300 python tools/knn_probe.py 1000000 768 64 bf16 64
timeout 900 python tools/index_bench.py 1000000 768 8 --modes exact,bf16 --recall
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc2 -c 1 -o gpurun_out/knn_tc2_1m64 python tools/knn_probe.py 1000000 768 8 bf16 64 > gpurun_out/ncu_tc2_1m64.log 2>&1; tail -3 gpurun_out/ncu_tc2_1m64.log
