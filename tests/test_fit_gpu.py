"""fit() end to end on the B200 (optimizer.hpp:327-482) against the
reference / oracle, and the GPU PCA initialisation (pca.hpp:79-218)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pipeline(O, x, C, W, epochs, seed):
    from oracle import train_config
    c = O.lsh_init(x, C, seed)
    c = O.kmeans_em(x, c, 100, O.default_kmeans_tol(x))
    g = O.build_knn(x, c, 15)
    pca = O.pca_init(x, seed)
    cfg = train_config(epochs=epochs, workers=W, seed=seed, n_clusters=C)
    lay, loss, means, _ = O.train_epochs(c.assignment, C, g.offsets, g.neighbors, 15, cfg, pca)
    return c, g, pca, lay, loss


def test_fit_bit_exact_with_injected_pca(port, ctx):
    """Replay-mode fit with the reference's PCA layout injected reproduces the
    reference's fit bit for bit (clusters, graph, layout)."""
    import paper_2505_15511_b200 as nb
    x = port.gaussian_mixture(3000, 24, 8, 10.0, 17)
    c, g, pca, lay, loss = _pipeline(port, x, 6, 3, 8, 5)
    rep = nb.FitReport()
    cfg = nb.TrainConfig(epochs=8, workers=3, seed=5, n_clusters=6)
    out = nb.fit(x, cfg, init_layout=pca, report=rep, ctx=ctx)
    assert np.array_equal(rep.clusters.assignment, c.assignment)
    assert np.array_equal(rep.graph.neighbors, g.neighbors)
    assert np.array_equal(rep.graph.distances, g.distances)
    assert np.array_equal(out, lay)
    np.testing.assert_allclose(rep.epoch_mean_loss, loss, rtol=1e-13, atol=0)


def test_fit_epochs_zero_returns_init(port, ctx):
    import paper_2505_15511_b200 as nb
    x = port.gaussian_mixture(800, 10, 4, 10.0, 3)
    pca = port.pca_init(x, 1)
    out = nb.fit(x, nb.TrainConfig(epochs=0, workers=2, seed=1, n_clusters=4), init_layout=pca,
                 ctx=ctx)
    assert np.array_equal(out, pca)


@pytest.mark.parametrize("n,d,blobs", [(3000, 24, 8), (2000, 200, 5), (700, 33, 3)])
def test_gpu_pca_bit_exact(port, ctx, n, d, blobs):
    """GPU PCA follows the reference's summation order in every data pass."""
    import paper_2505_15511_b200 as nb
    x = port.gaussian_mixture(n, d, blobs, 10.0, 23)
    ref = port.pca_init(x, 9)
    got = nb.pca_init(x, 9, ctx=ctx)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("n,d,blobs", [(3000, 24, 8), (2000, 200, 5), (700, 33, 3)])
def test_gpu_pca_fast_tolerance(port, ctx, n, d, blobs):
    """Precomputed-covariance PCA: same algorithm, covariance formed once. The
    layout spans the reference's principal plane (its columns are linear
    combinations of the reference's); the in-plane orientation is fixed by
    the reference's Rayleigh-Ritz rotation, whose angle is computed from
    rounding noise once the basis has converged (pca.hpp:150-165)."""
    import paper_2505_15511_b200 as nb
    x = port.gaussian_mixture(n, d, blobs, 10.0, 23)
    ref = port.pca_init(x, 9)
    got = nb.pca_init(x, 9, ctx=ctx, fast=True)
    coef, *_ = np.linalg.lstsq(ref, got, rcond=None)
    assert np.abs(got - ref @ coef).max() < 1e-8
    np.testing.assert_allclose(got.mean(0), 0, atol=1e-9)
    np.testing.assert_allclose(got.std(0), 1, atol=1e-9)


def test_gpu_pca_fast_rank_one_jitter(port, ctx):
    import paper_2505_15511_b200 as nb
    t = np.linspace(-1, 1, 500)
    x = np.ascontiguousarray(np.outer(t, np.arange(1, 9)).astype(np.float32))
    ref = port.pca_init(x, 4)
    got = nb.pca_init(x, 4, ctx=ctx, fast=True)
    np.testing.assert_allclose(got[:, 0], ref[:, 0], rtol=0, atol=1e-9)
    assert np.array_equal(got[:, 1], ref[:, 1])  # the seeded jitter


def test_fit_fully_on_gpu_is_bit_exact(port, ref, ctx):
    """The whole fit() on the GPU (LSH k-means, certified kNN, PCA, replay
    epochs) reproduces the reference's fit() bit for bit."""
    import paper_2505_15511_b200 as nb
    from oracle import train_config
    x = port.gaussian_mixture(2500, 20, 6, 10.0, 31)
    kw = dict(epochs=12, workers=2, n_clusters=5)
    r = ref.fit(x, train_config(seed=3, **kw))
    rep = nb.FitReport()
    out = nb.fit(x, nb.TrainConfig(seed=3, **kw), report=rep, ctx=ctx)
    assert np.array_equal(out, r["layout"])
    np.testing.assert_allclose(rep.epoch_mean_loss, r["epoch_loss"], rtol=1e-13, atol=0)
    # FitReport (optimizer.hpp:312-321), every field from the engine's outputs
    assert np.array_equal(rep.clusters.assignment, r["assignment"])
    assert np.array_equal(rep.graph.offsets, r["offsets"])
    assert np.array_equal(rep.graph.neighbors, r["neighbors"])
    assert np.array_equal(rep.graph.distances, r["distances"])
    assert np.array_equal(rep.pca, r["pca"])
    assert np.array_equal(rep.final_means, r["final_means"])
    cnt = np.diff(rep.graph.offsets.astype(np.int64))
    want = np.concatenate([ref.inverse_rank_weights(int(c)) for c in cnt if c > 0])
    assert np.array_equal(rep.affinity.weights, want)  # affinity.hpp:65-84
    assert np.array_equal(rep.affinity.eligible_heads, np.nonzero(cnt)[0])
    c2w, wpts = ref.shard_clusters(r["assignment"], r["n_clusters"], kw["workers"])
    assert np.array_equal(rep.plan.cluster_to_worker, c2w)
    assert all(np.array_equal(a, b) for a, b in zip(rep.plan.worker_points, wpts))
    assert (rep.comm.epochs, rep.comm.messages) == (12, 12 * 2)


def test_gpu_pca_rank_one_jitter(port, ctx):
    """Rank-1 data: second coordinate is the reference's seeded jitter."""
    import paper_2505_15511_b200 as nb
    t = np.linspace(-1, 1, 500)
    x = np.ascontiguousarray(np.outer(t, np.arange(1, 9)).astype(np.float32))
    ref = port.pca_init(x, 4)
    got = nb.pca_init(x, 4, ctx=ctx)
    assert np.array_equal(got, ref)


def test_gpu_pca_degenerate(ctx):
    import paper_2505_15511_b200 as nb
    with pytest.raises(nb.NomadError) as e:
        nb.pca_init(np.ones((20, 3), np.float32), ctx=ctx)
    assert e.value.kind == "Degenerate"


def test_fit_with_gpu_pca_quality(port, ctx):
    """Full GPU fit (GPU PCA, throughput SGD): loss trajectory tracks the
    reference's within 5% after 40 epochs."""
    import paper_2505_15511_b200 as nb
    x = port.gaussian_mixture(4000, 32, 10, 10.0, 42)
    *_, rloss = _pipeline(port, x, 5, 1, 40, 7)
    rep = nb.FitReport()
    out = nb.fit(x, nb.TrainConfig(epochs=40, workers=1, seed=7, n_clusters=5,
                                   sgd_mode="hogwild"), report=rep, ctx=ctx)
    assert np.isfinite(out).all()
    l = np.array(rep.epoch_mean_loss)
    assert abs(l[-5:].mean() - rloss[-5:].mean()) < 0.05 * rloss[-5:].mean()


@pytest.mark.parametrize("n,d", [(3000, 24), (2000, 200), (700, 33), (50000, 768)])
def test_covariance_sums(ctx, n, d):
    """The fast PCA's covariance pass against numpy fp64."""
    import ctypes as C
    import paper_2505_15511_b200 as nb
    from paper_2505_15511_b200 import _native as N
    from paper_2505_15511_b200.api import _dataset
    x = np.random.default_rng(n).normal(size=(n, d)).astype(np.float32) * 3 + 1
    m = x.astype(np.float64).mean(0)
    out = np.zeros((d, d))
    dv, keep = _dataset(x)
    N.check(nb.lib().nomad_b200_debug_cov(ctx.h, C.byref(dv), m.ctypes.data, out.ctypes.data))
    xc = x.astype(np.float64) - m
    np.testing.assert_allclose(out, xc.T @ xc, rtol=1e-11, atol=1e-9 * n)
