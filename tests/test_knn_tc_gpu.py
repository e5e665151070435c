"""bf16 tcgen05 kNN fast mode: the raw TMA + tcgen05.mma + TMEM tile product,
and recall@k of the fast graph against the exact graph."""
import ctypes as C

import numpy as np
import pytest

from common import index_case

pytestmark = pytest.mark.gpu


def _bf16(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)  # RNE
    return r.view(np.float32)


@pytest.mark.parametrize("fp16", [False, True])
@pytest.mark.parametrize("d", [64, 192, 768, 100])
def test_tc_tile_gemm_matches_numpy(ctx, d, fp16):
    import paper_2505_15511_b200 as nb
    rng = np.random.default_rng(d)
    x = rng.normal(size=(384, d)).astype(np.float32)
    out = np.zeros((128, 128), np.float32)
    a0 = 0x80000000 if fp16 else 0
    nb._native.check(nb.lib().nomad_b200_debug_tc_gemm(ctx.h, x.ctypes.data, 384, d, a0, 256,
                                                       out.ctypes.data))
    xb = (x.astype(np.float16).astype(np.float64) if fp16 else _bf16(x).astype(np.float64))
    ref = xb[0:128] @ xb[256:384].T
    np.testing.assert_allclose(out, ref, rtol=1e-4, atol=1e-3 * np.sqrt(d))


@pytest.mark.parametrize("n,d,blobs,C", [(3000, 32, 10, 8), (2500, 768, 8, 4), (5000, 100, 5, 6)])
def test_bf16_knn_recall(port, ctx, n, d, blobs, C):
    import paper_2505_15511_b200 as nb
    x, c, g, _ = index_case(n, d, blobs, C, 15)
    ca = nb.ClusterAssignment(c.assignment, c.n_clusters, d, c.centroids, c.sizes)
    fast = nb.build_knn(x, ca, 15, mode="bf16", ctx=ctx)
    assert np.array_equal(fast.offsets, g.offsets)
    hits = 0
    for i in range(n):
        a = set(g.neighbors[g.offsets[i]:g.offsets[i + 1]].tolist())
        b = fast.neighbors[fast.offsets[i]:fast.offsets[i + 1]]
        hits += len(a.intersection(b.tolist()))
        # reported distances are the exact fp64 ones, ascending by (dist, id)
        dd = fast.distances[fast.offsets[i]:fast.offsets[i + 1]]
        assert np.all(np.diff(dd) >= 0)
    recall = hits / len(g.neighbors)
    assert recall >= 0.95, recall
