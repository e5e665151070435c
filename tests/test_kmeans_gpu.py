"""k-means partitioner parity on the B200 (kmeans.hpp:47-296): assignments,
centroids, sizes and the quantisation-error trace are bit-identical to the
oracle (and, through tests/golden, to the reference)."""
import json
import os

import numpy as np
import pytest

from common import sha

pytestmark = pytest.mark.gpu
G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_goldens.json")))


def _eq(a, b):
    return np.array_equal(np.asarray(a), np.asarray(b))


@pytest.mark.parametrize("n,d,blobs,C,seed", [(3000, 32, 10, 8, 7), (5000, 17, 6, 13, 3),
                                              (2000, 48, 3, 40, 11)])
def test_lsh_kmeans_bit_exact(port, ctx, n, d, blobs, C, seed):
    import paper_2505_15511_b200 as nb
    x = port.gaussian_mixture(n, d, blobs, 10.0, 42 + seed)
    r0 = port.lsh_init(x, C, seed)
    g0 = nb.lsh_init(x, C, seed, ctx=ctx)
    assert _eq(g0.assignment, r0.assignment) and _eq(g0.sizes, r0.sizes)
    assert _eq(g0.centroids, r0.centroids)
    tol = port.default_kmeans_tol(x)
    assert nb.default_kmeans_tol(x, ctx=ctx) == tol
    r1, rqe = port.kmeans_em(x, r0, 100, tol, trace=True)
    qe = []
    g1 = nb.kmeans_em(x, g0, 100, tol, qe_trace=qe, ctx=ctx)
    assert _eq(g1.assignment, r1.assignment) and _eq(g1.sizes, r1.sizes)
    assert _eq(g1.centroids, r1.centroids)
    assert _eq(qe, rqe)
    g2 = nb.kmeans_em_default_tol(x, g0, 100, ctx=ctx)
    assert _eq(g2.assignment, r1.assignment) and _eq(g2.centroids, r1.centroids)


def test_lsh_perturbation_and_repair(port, ctx):
    """Few distinct points: fewer non-empty buckets than clusters triggers the
    perturbation branch (kmeans.hpp:228-242) and empty-cluster repair
    (:109-143)."""
    import paper_2505_15511_b200 as nb
    base = port.gaussian_mixture(4, 6, 4, 10.0, 5)
    x = np.ascontiguousarray(np.repeat(base, 30, axis=0))
    for C in (5, 9):
        r0 = port.lsh_init(x, C, 1)
        g0 = nb.lsh_init(x, C, 1, ctx=ctx)
        assert _eq(g0.assignment, r0.assignment) and _eq(g0.centroids, r0.centroids)
        assert _eq(g0.sizes, r0.sizes)
        r1 = port.kmeans_em(x, r0, 20, 0.0)
        g1 = nb.kmeans_em(x, g0, 20, 0.0, ctx=ctx)
        assert _eq(g1.assignment, r1.assignment) and _eq(g1.centroids, r1.centroids)


@pytest.mark.parametrize("case", ["small_w4", "config_a_w1"])
def test_kmeans_matches_reference_goldens(port, ctx, case):
    import paper_2505_15511_b200 as nb
    gc = G["cases"][case]
    n, d, blobs, ncl = gc["shape"][:4]
    x = port.gaussian_mixture(n, d, blobs, 10.0, 42)
    g0 = nb.lsh_init(x, ncl, 7, ctx=ctx)
    assert sha(g0.assignment) == gc["lsh_assignment"]
    assert sha(g0.centroids) == gc["lsh_centroids"]
    qe = []
    g1 = nb.kmeans_em_default_tol(x, g0, 100, qe_trace=qe, ctx=ctx)
    assert sha(g1.assignment) == gc["km_assignment"]
    assert sha(g1.centroids) == gc["km_centroids"]
    assert [float(v).hex() for v in qe] == gc["qe_trace"]


def test_kmeans_errors(ctx):
    import paper_2505_15511_b200 as nb
    x = np.random.default_rng(0).normal(size=(50, 4)).astype(np.float32)
    with pytest.raises(nb.NomadError) as e:
        nb.lsh_init(x, 1, 0, ctx=ctx)
    assert e.value.kind == "Parameter" and "cluster count must be in [2, n]" in e.value.message
    with pytest.raises(nb.NomadError) as e:
        nb.lsh_init(x, 51, 0, ctx=ctx)
    assert e.value.kind == "Parameter"
