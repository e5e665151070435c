"""Exact kNN build at 10M x 768 (C=64), repeated in one process, with per-stage timing
(NOMAD_B200_DEBUG_KNN=1) and the SM clock sampled by NVML around each build."""
import sys
import threading
import time
sys.path.insert(0, ".")
import pynvml  # noqa: E402
import torch  # noqa: E402
import paper_2505_15511_b200 as nb  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
ctx = nb.Context(0)
x = nb.generate_mixture(10_000_000, 768, 64, 10.0, 42, ctx=ctx)
c = nb.kmeans_em_default_tol(x, nb.lsh_init(x, 64, 7, ctx=ctx), 100, ctx=ctx)
for rep in range(4):
    clk, stop = [], [False]
    def sample():
        while not stop[0]:
            clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            time.sleep(0.05)
    th = threading.Thread(target=sample)
    th.start()
    torch.cuda.synchronize()
    t = time.perf_counter()
    nb.build_knn(x, c, 15, mode="exact", ctx=ctx)
    dt = time.perf_counter() - t
    stop[0] = True
    th.join()
    clk.sort()
    print(f"rep {rep}: {dt:.2f} s, SM clock min/median/max {clk[0]}/{clk[len(clk)//2]}/{clk[-1]} MHz",
          file=sys.stderr, flush=True)
