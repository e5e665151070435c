timeout 900 python -m pytest tests/test_knn_gpu.py tests/test_scale_gpu.py -x -q --timeout 600 2>&1 | tail -5
timeout 300 python tools/knn_probe.py 40000 768 2 exact_ffma
timeout 300 python tools/knn_probe.py 40000 768 2 exact
timeout 600 python tools/index_bench.py 1000000 768 8 --modes exact,exact_ffma,bf16
