"""Device->host copy rates into the kinds of host memory build_knn writes:
fresh calloc'd numpy (np.zeros, first touch during the copy), pre-faulted
numpy, pinned. python tools/d2h_probe.py [GB]"""
import sys
import time

import numpy as np
import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 1.8
n = int(gb * 2**30 / 8)
t = torch.ones(n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def timed(what, dst):
    torch.cuda.synchronize()
    a = time.perf_counter()
    dst.copy_(t)
    torch.cuda.synchronize()
    s = time.perf_counter() - a
    print(f"{what:34s} {s*1e3:8.1f} ms  {n*8/s/1e9:6.1f} GB/s")


timed("np.zeros (first touch)", torch.from_numpy(np.zeros(n)))
a = np.zeros(n)
a[:] = 1.0
timed("np pre-faulted", torch.from_numpy(a))
timed("pinned", torch.empty(n, dtype=torch.float64, pin_memory=True))
a = time.perf_counter()
z = np.zeros(n)
z[::512] = 1.0
print(f"{'first-touch fault cost (1 thread)':34s} {(time.perf_counter()-a)*1e3:8.1f} ms")
