cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 red_bench.cu -o red_bench && timeout 120 ./red_bench; cd ../..
timeout 300 python tools/knn_probe.py 1000000 768 8 bf16 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_knn_tc2 -c 1 -o gpurun_out/knn_tc2_1m python tools/knn_probe.py 1000000 768 8 bf16 > gpurun_out/ncu_tc2_1m.log 2>&1; tail -3 gpurun_out/ncu_tc2_1m.log
