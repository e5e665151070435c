timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -5
timeout 300 python tools/index_bench.py 1000000 768 8 --modes bf16
timeout 300 python tools/index_bench.py 1000000 768 8 --modes bf16,bf16
timeout 600 python tools/index_bench.py 1000000 768 8 --modes exact_ffma,exact
