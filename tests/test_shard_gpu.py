"""Row-sharded index build: G ranks each holding only a slice
of the rows (a loopback group on one B200 runs the same per-rank code and
collectives' data flow as G GPUs). LSH init and Lloyd iterations with the
ascending-id sums carried rank to rank, the rows' all-to-all to their cluster
owners and the per-rank kNN build must reproduce the one-GPU index bit for
bit — which is itself the reference's (test_kmeans_gpu.py, test_knn_gpu.py) —
and the sharded graph must train to the oracle's replay trajectory."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _slices(n, G, rng):
    cuts = np.sort(rng.choice(np.arange(1, n), size=G - 1, replace=False))
    b = np.concatenate([[0], cuts, [n]])
    return [(int(b[r]), int(b[r + 1] - b[r])) for r in range(G)]


@pytest.mark.parametrize("G,dtype,mode", [(2, "f32", "exact"), (3, "f32", "exact"),
                                          (4, "bf16", "exact"), (4, "f32", "bf16")])
def test_sharded_index_equals_one_gpu(ctx, G, dtype, mode):
    import torch
    import paper_2505_15511_b200 as nb
    n, d, blobs, C, W = 6000, 32, 10, 8, 2 * G
    x = nb.generate_mixture(n, d, blobs, 10.0, 42, ctx=ctx, dtype=dtype)
    c1 = nb.kmeans_em_default_tol(x, nb.lsh_init(x, C, 7, ctx=ctx), 100, ctx=ctx)
    g1 = nb.build_knn(x, c1, 15, mode=mode, ctx=ctx)
    grp = nb.Group([0] * G)
    sl = _slices(n, G, np.random.default_rng(G))
    rows = [nb.generate_mixture_rows(r0, m, d, blobs, 10.0, 42, ctx=grp.context(r), dtype=dtype)
            for r, (r0, m) in enumerate(sl)]
    for r, (r0, m) in enumerate(sl):  # the row slices are the full matrix's rows
        assert torch.equal(rows[r], x[r0:r0 + m])
    cs, gs = nb.group_index_sharded(grp, rows, [r0 for r0, _ in sl], n, C, 7, W, 15,
                                    knn_mode=mode)
    assert np.array_equal(cs.assignment, c1.assignment)
    assert np.array_equal(cs.centroids, c1.centroids)
    assert np.array_equal(cs.sizes, c1.sizes)
    assert np.array_equal(gs.offsets, g1.offsets)
    assert np.array_equal(gs.neighbors, g1.neighbors)
    assert np.array_equal(gs.distances, g1.distances)


def test_sharded_index_trains_to_the_oracle(port):
    """Sharded index over 4 ranks -> replay epochs over the same 4 ranks: the
    reference's trajectory (clusters may be split between ranks' rows, each
    cluster's rows gathered on its owner)."""
    import paper_2505_15511_b200 as nb
    from common import index_case
    from oracle import train_config
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    grp = nb.Group([0] * 4)
    sl = [(0, 700), (700, 900), (1600, 500), (2100, 900)]
    import torch
    xt = torch.from_numpy(x).cuda()
    cs, gs = nb.group_index_sharded(grp, [xt[a:a + m] for a, m in sl], [a for a, _ in sl], 3000,
                                    8, 7, 8, 15)
    assert np.array_equal(cs.assignment, c.assignment)
    assert np.array_equal(gs.neighbors, g.neighbors) and np.array_equal(gs.distances, g.distances)
    kw = dict(epochs=10, workers=8, seed=7)
    tr = nb.Trainer(gs, cs, pca, nb.TrainConfig(**kw), group=grp)
    loss = tr.run(3)
    rl, rloss, _, _ = port.train_epochs(c.assignment, c.n_clusters, g.offsets, g.neighbors, 15,
                                        train_config(**kw), pca, 0, 3)
    assert np.array_equal(tr.layout(), rl)
    np.testing.assert_allclose(loss, rloss, rtol=1e-13, atol=0)


def test_single_rank_sharded_build(ctx):
    """nomad_b200_index_sharded with world_size 1 (the multi-process entry on one
    rank) is the one-GPU build."""
    import paper_2505_15511_b200 as nb
    n, d, blobs, C = 5000, 24, 8, 6
    x = nb.generate_mixture(n, d, blobs, 10.0, 3, ctx=ctx)
    c1 = nb.kmeans_em_default_tol(x, nb.lsh_init(x, C, 5, ctx=ctx), 100, ctx=ctx)
    g1 = nb.build_knn(x, c1, 15, ctx=ctx)
    cs, gs = nb.index_sharded(x, 0, n, C, 5, 2, k=15, ctx=ctx)
    assert np.array_equal(cs.assignment, c1.assignment)
    assert np.array_equal(cs.centroids, c1.centroids)
    assert np.array_equal(gs.neighbors, g1.neighbors) and np.array_equal(gs.distances, g1.distances)
