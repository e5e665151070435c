"""Wall time of build_knn into host numpy (the API call) per mode, at config C
scale: python tools/knn_wall.py [N] [C]"""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2505_15511_b200 as nb  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
C = int(sys.argv[2]) if len(sys.argv) > 2 else 64
ctx = nb.Context(0)
x = nb.generate_mixture(n, 768, 64, 10.0, 42, ctx=ctx)
c = nb.kmeans_em_default_tol(x, nb.lsh_init(x, C, 7, ctx=ctx), 100, ctx=ctx)
for mode in ["exact", "bf16", "exact", "bf16"]:
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = nb.build_knn(x, c, 15, mode=mode, ctx=ctx)
    print(f"{mode:6s} {time.perf_counter() - t:6.2f} s", flush=True)
    del g
