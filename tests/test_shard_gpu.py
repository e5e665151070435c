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


@pytest.mark.parametrize("G,dtype", [(2, "f32"), (3, "f32"), (4, "bf16")])
def test_sharded_pca_exact_equals_one_gpu(ctx, G, dtype):
    """Row-sharded pca_init: the data mean, every covariance
    apply's column chains and the layout's column mean / spread carried rank
    to rank -> the one-GPU (= reference, test_fit_gpu.py) layout bit for bit."""
    import torch
    import paper_2505_15511_b200 as nb
    n, d = 5000, 24
    x = nb.generate_mixture(n, d, 6, 10.0, 5, ctx=ctx, dtype=dtype)
    one = nb.pca_init(x, seed=3, ctx=ctx)
    grp = nb.Group([0] * G)
    sl = _slices(n, G, np.random.default_rng(10 + G))
    rows = [x[a:a + m] for a, m in sl]
    parts = nb.group_pca_init_sharded(grp, rows, [a for a, _ in sl], n, seed=3)
    assert np.array_equal(np.concatenate(parts), one)
    torch.cuda.synchronize()


def test_sharded_pca_rank_deficient_jitter(ctx):
    """Rank-1 data: the second component is the reference's uniform jitter
    (pca.hpp:189-195), drawn in row order — every rank skips the draws of
    the rows before its slice."""
    import torch
    import paper_2505_15511_b200 as nb
    rng = np.random.default_rng(4)
    n, d = 3000, 16
    x = np.outer(rng.normal(size=n), rng.normal(size=d)).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    one = nb.pca_init(xt, seed=9, ctx=ctx)
    grp = nb.Group([0] * 3)
    sl = [(0, 1000), (1000, 700), (1700, 1300)]
    parts = nb.group_pca_init_sharded(grp, [xt[a:a + m] for a, m in sl], [a for a, _ in sl], n,
                                      seed=9)
    assert np.array_equal(np.concatenate(parts), one)


def test_sharded_pca_fast_same_plane(ctx):
    """fast=True: the ranks' covariance sums added in rank order give the
    one-GPU fast form's principal plane (orientation inside the plane is
    rounding-level, pca.cu)."""
    import paper_2505_15511_b200 as nb
    n, d = 8000, 32
    x = nb.generate_mixture(n, d, 8, 10.0, 6, ctx=ctx)
    one = nb.pca_init(x, seed=1, ctx=ctx, fast=True)
    grp = nb.Group([0] * 2)
    parts = nb.group_pca_init_sharded(grp, [x[:3000], x[3000:]], [0, 3000], n, seed=1, fast=True)
    two = np.concatenate(parts)
    # both standardised: the same plane <=> Y1^T Y2 / n is orthogonal
    m = one.T @ two / n
    sv = np.linalg.svd(m, compute_uv=False)
    np.testing.assert_allclose(sv, [1.0, 1.0], atol=1e-6)
