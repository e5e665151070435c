"""Exact kNN graph parity on the B200 (knn.hpp:51-109): neighbour ids AND
fp64 distances bit-identical to the oracle / reference goldens, including
ragged lists, singleton clusters and massive ties (certificate fallback)."""
import json
import os

import numpy as np
import pytest

from common import sha, index_case

pytestmark = pytest.mark.gpu
G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_goldens.json")))


def _gpu_graph(nb, ctx, x, c, k, mode="exact"):
    ca = nb.ClusterAssignment(c.assignment, c.n_clusters, x.shape[1], c.centroids, c.sizes)
    return nb.build_knn(x, ca, k, mode=mode, ctx=ctx)

MODES = ["exact", "exact_ffma"]  # tensor-core certified filter / FFMA certified filter


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("n,d,blobs,C,k", [(3000, 32, 10, 8, 15), (600, 8, 40, 40, 15),
                                           (4000, 100, 5, 6, 7), (2500, 768, 8, 4, 15),
                                           (3000, 50, 6, 5, 40)])
def test_knn_bit_exact(port, ctx, n, d, blobs, C, k, mode):
    import paper_2505_15511_b200 as nb
    x, c, g, _ = index_case(n, d, blobs, C, k)
    gg = _gpu_graph(nb, ctx, x, c, k, mode)
    assert np.array_equal(gg.offsets, g.offsets)
    assert np.array_equal(gg.neighbors, g.neighbors)
    assert np.array_equal(gg.distances, g.distances)


@pytest.mark.parametrize("mode", MODES)
def test_knn_ties_and_singletons(port, ctx, mode):
    """Exact duplicates make every k-th distance a tie at 0 (the certificate
    cannot hold, so the exhaustive fp64 path decides by id), plus clusters of
    size 1 (empty lists) and 2."""
    import paper_2505_15511_b200 as nb
    from oracle import Clusters
    base = port.gaussian_mixture(40, 12, 4, 10.0, 9)
    x = np.ascontiguousarray(np.repeat(base, 50, axis=0))
    a = (np.arange(len(x)) % 3).astype(np.uint32)
    a[0] = 3            # singleton
    a[1] = a[2] = 4     # pair
    cl = Clusters(a, np.zeros(5), np.bincount(a, minlength=5).astype(np.uint32), 5, 12)
    g = port.build_knn(x, cl, 15)
    gg = _gpu_graph(nb, ctx, x, cl, 15, mode)
    assert np.array_equal(gg.offsets, g.offsets)
    assert np.array_equal(gg.neighbors, g.neighbors)
    assert np.array_equal(gg.distances, g.distances)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("case", ["small_w4", "config_a_w1"])
def test_knn_matches_reference_goldens(port, ctx, case, mode):
    """Whole GPU index build (lsh_init -> kmeans_em -> build_knn) vs the
    reference's outputs on the golden inputs."""
    import paper_2505_15511_b200 as nb
    gc = G["cases"][case]
    n, d, blobs, ncl, k = gc["shape"][:5]
    x = port.gaussian_mixture(n, d, blobs, 10.0, 42)
    c = nb.kmeans_em_default_tol(x, nb.lsh_init(x, ncl, 7, ctx=ctx), 100, ctx=ctx)
    gg = nb.build_knn(x, c, k, mode=mode, ctx=ctx)
    assert sha(gg.offsets) == gc["knn_offsets"]
    assert sha(gg.neighbors) == gc["knn_neighbors"]
    assert sha(gg.distances) == gc["knn_distances"]


@pytest.mark.parametrize("d", [64, 50])
def test_knn_multiblob_clusters_open_rows(port, ctx, d):
    """Clusters that merge far-apart blobs: large centred norms leave many rows
    uncertified by the fp16 tensor-core filter; those rows (only) are
    re-filtered by the FFMA kernel (d % 4 == 0: pipelined query-list form;
    otherwise the scalar whole-cluster form) and the result is still
    bit-identical to the oracle."""
    import paper_2505_15511_b200 as nb
    from oracle import Clusters
    x = port.gaussian_mixture(8000, d, 24, 60.0, 3)
    a = (np.arange(len(x)) % 2).astype(np.uint32)  # every cluster spans all blobs
    cl = Clusters(a, np.zeros(2 * d), np.bincount(a, minlength=2).astype(np.uint32), 2, d)
    g = port.build_knn(x, cl, 15)
    gg = _gpu_graph(nb, ctx, x, cl, 15, "exact")
    tc_open, _ = ctx.knn_stats()
    assert tc_open > 0
    assert np.array_equal(gg.offsets, g.offsets)
    assert np.array_equal(gg.neighbors, g.neighbors)
    assert np.array_equal(gg.distances, g.distances)


@pytest.mark.parametrize("mode", ["exact", "bf16"])
def test_knn_shard_owned_clusters(port, ctx, mode):
    """Multi-GPU index build: lists only for the owned clusters (a rank's
    shards), identical to the full build there, empty elsewhere."""
    import paper_2505_15511_b200 as nb
    x, c, g, _ = index_case(3000, 32, 10, 8, 15)
    ca = nb.ClusterAssignment(c.assignment, c.n_clusters, x.shape[1], c.centroids, c.sizes)
    full = nb.build_knn(x, ca, 15, mode=mode, ctx=ctx)
    c2w, _ = nb.shard_plan(c.assignment, c.n_clusters, 4, 2)
    owned = np.nonzero(c2w >= 2)[0]  # rank 1 of 2 (workers 2, 3)
    part = nb.build_knn(x, ca, 15, mode=mode, ctx=ctx, owned_clusters=owned)
    mine = np.isin(c.assignment, owned)
    cnt_full = np.diff(full.offsets.astype(np.int64))
    cnt_part = np.diff(part.offsets.astype(np.int64))
    assert np.array_equal(cnt_part, np.where(mine, cnt_full, 0))
    for i in np.nonzero(mine)[0][:500]:
        assert np.array_equal(part.neighbors_of(i), full.neighbors_of(i))
    assert nb.build_knn(x, ca, 15, mode=mode, ctx=ctx, owned_clusters=[]).offsets[-1] == 0


def test_knn_subcluster_stage_certifies_blobs(port, ctx):
    """One cluster holding three far-apart blobs: the fp16 certificate on the
    cluster's centring fails, the sub-cluster stage (bisection into the
    blobs, certified tensor-core lists inside each, geometric bound across)
    settles almost every row; the graph is still bit-identical."""
    import paper_2505_15511_b200 as nb
    from oracle import Clusters
    x = port.gaussian_mixture(9000, 48, 3, 60.0, 5)
    a = np.zeros(len(x), np.uint32)
    cl = Clusters(a, np.zeros(48), np.array([len(x)], np.uint32), 1, 48)
    g = port.build_knn(x, cl, 15)
    gg = _gpu_graph(nb, ctx, x, cl, 15, "exact")
    tc_open, _ = ctx.knn_stats()
    assert tc_open > 0.5 * len(x)
    assert ctx.knn_subcluster_rows() > 0.9 * tc_open
    assert np.array_equal(gg.offsets, g.offsets)
    assert np.array_equal(gg.neighbors, g.neighbors)
    assert np.array_equal(gg.distances, g.distances)
