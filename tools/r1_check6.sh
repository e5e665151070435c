timeout 300 python tools/pca_debug.py 2>&1 | grep -E "fast-exact"
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 600 2>&1 | tail -4
timeout 600 python -c "
import sys, time; sys.path.insert(0,'.')
import torch, paper_2505_15511_b200 as nb
ctx = nb.Context(0)
for n in (1000000, 10000000):
    x = nb.generate_mixture(n, 768, 64, 10.0, 42, ctx=ctx)
    torch.cuda.synchronize(); t = time.perf_counter()
    y = nb.pca_init(x, 7, ctx=ctx, fast=True)
    print('fast pca', n, round(time.perf_counter() - t, 2), 's', y[:2].tolist(), flush=True)
    del x
"
timeout 1500 python tools/quality_scale.py 1000000 768 64 8 200 8
