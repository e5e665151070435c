"""Break the bench's e2e path into its pieces (synthetic config C index)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2505_15511_b200 as nb  # noqa: E402

n, d, blobs, ncl, W = bench.CONFIGS["C"]
a, off, nbr, init = bench.synthetic_index(n, ncl, 15)
ctx = nb.Context(0)
tr = nb.Trainer(nb.KnnGraph(n, 15, off, nbr, np.zeros(0)),
                nb.ClusterAssignment(a, ncl, d, np.zeros(0), np.zeros(0)), init,
                nb.TrainConfig(epochs=200, workers=W, seed=7, sgd_mode="hogwild"), ctx=ctx)
tr.run(3)
hin = torch.from_numpy(init).pin_memory()
hout = torch.empty((n, 2), dtype=torch.float64).pin_memory()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); tr.set_layout(hin); t1 = time.perf_counter()
    tr.run(20); t2 = time.perf_counter()
    tr.layout(hout.numpy()); t3 = time.perf_counter()
    print(f"set_layout {1e3*(t1-t0):.1f} ms  run(20) {1e3*(t2-t1):.1f} ms  layout {1e3*(t3-t2):.1f} ms")
