"""Epoch loop parity on the B200: replay mode must be bit-identical to the
oracle (the C restatement of optimizer.hpp:232-470, itself pinned to the
reference in test_oracle.py); hogwild mode must match statistically."""
import numpy as np
import pytest

from common import index_case

pytestmark = pytest.mark.gpu


def _trainer(nb, ctx, c, g, pca, **kw):
    cfg = nb.TrainConfig(**kw)
    return nb.Trainer(nb.KnnGraph(len(c.assignment), g.k, g.offsets, g.neighbors, g.distances),
                      nb.ClusterAssignment(c.assignment, c.n_clusters, c.dims, c.centroids,
                                           c.sizes), pca, cfg, ctx=ctx)


def _oracle(port, c, g, pca, n_run, **kw):
    from oracle import train_config
    return port.train_epochs(c.assignment, c.n_clusters, g.offsets, g.neighbors, g.k,
                             train_config(**kw), pca, 0, n_run)


@pytest.mark.parametrize("workers", [1, 4])
def test_replay_bit_exact(port, ctx, workers):
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=10, workers=workers, seed=7)
    tr = _trainer(nb, ctx, c, g, pca, **kw)
    loss = tr.run(6)
    lay = tr.layout()
    rl, rloss, rmeans, _ = _oracle(port, c, g, pca, 6, **kw)
    assert np.array_equal(lay, rl)
    # loss goes through CUDA's log (<= 1 ulp from glibc): relative 1e-13
    np.testing.assert_allclose(loss, rloss, rtol=1e-13, atol=0)
    m, counts = tr.means()
    assert np.array_equal(m, rmeans)
    assert counts.tolist() == c.sizes.tolist()
    log = tr.comm_log()
    assert (log.epochs, log.messages) == (6, 6 * workers)
    assert log.payload_doubles == 6 * 2 * 8 and log.payload_counts == 6 * 8


@pytest.mark.parametrize("k,s", [(40, 5), (20, 14)])
def test_replay_long_touch_lists(port, ctx, k, s):
    """1 + k + s > 32 slots per draw: the per-thread dataflow form (and touch
    rows wider than a warp) must stay bit-identical too."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(2000, 16, 10, 8, k)
    kw = dict(epochs=10, workers=4, seed=11, k=k, local_draws=s)
    tr = _trainer(nb, ctx, c, g, pca, **kw)
    loss = tr.run(3)
    rl, rloss, _, _ = _oracle(port, c, g, pca, 3, **kw)
    assert np.array_equal(tr.layout(), rl)
    np.testing.assert_allclose(loss, rloss, rtol=1e-13, atol=0)


def test_replay_host_draw_fallback_is_identical(port, ctx, monkeypatch):
    """The rejection branch of uniform_index (rng.hpp:49-55, probability
    ~n / 2^64 per draw) moves a worker's draws to the host for that epoch;
    forced for every epoch and worker, the run must stay bit-identical."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=10, workers=4, seed=7)
    monkeypatch.setenv("NOMAD_B200_REPLAY_HOST_DRAWS", "1")
    tr = _trainer(nb, ctx, c, g, pca, **kw)
    loss = tr.run(3)
    monkeypatch.delenv("NOMAD_B200_REPLAY_HOST_DRAWS")
    loss2 = tr.run(2)
    rl, rloss, _, _ = _oracle(port, c, g, pca, 5, **kw)
    assert np.array_equal(tr.layout(), rl)
    np.testing.assert_allclose(np.concatenate([loss, loss2]), rloss, rtol=1e-13, atol=0)


def test_replay_repeated_list_entries(port, ctx):
    """A caller's graph may repeat a neighbour inside a list (the reference then
    applies both updates in turn); the dependency lists must not make the
    draw wait on itself."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    nbr = g.neighbors.copy().reshape(-1, 15)
    nbr[::7, 3] = nbr[::7, 1]
    nbr[::11, 14] = nbr[::11, 0]
    kw = dict(epochs=10, workers=4, seed=7)
    tr = nb.Trainer(nb.KnnGraph(3000, 15, g.offsets, nbr.reshape(-1), g.distances),
                    nb.ClusterAssignment(c.assignment, c.n_clusters, c.dims, c.centroids, c.sizes),
                    pca, nb.TrainConfig(**kw), ctx=ctx)
    loss = tr.run(3)
    from oracle import train_config
    rl, rloss, _, _ = port.train_epochs(c.assignment, c.n_clusters, g.offsets, nbr.reshape(-1), 15,
                                        train_config(**kw), pca, 0, 3)
    assert np.array_equal(tr.layout(), rl)
    np.testing.assert_allclose(loss, rloss, rtol=1e-13, atol=0)


def test_replay_resume_equals_single_run(port, ctx):
    """run(2)+run(3) == run(5): worker RNG streams persist across calls."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=8, workers=2, seed=3)
    a = _trainer(nb, ctx, c, g, pca, **kw)
    a.run(2)
    a.run(3)
    b = _trainer(nb, ctx, c, g, pca, **kw)
    b.run(5)
    assert np.array_equal(a.layout(), b.layout())


@pytest.mark.parametrize("mode", ["all_but_own", "head_only"])
def test_replay_ablation_modes(port, ctx, mode):
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=10, workers=2, seed=11)
    okw = dict(kw)
    if mode == "all_but_own":
        kw["approx"] = "non-own-cluster"
        okw["approx_all_but_own"] = 1
    else:
        kw["head_only"] = True
        okw["head_only"] = 1
    tr = _trainer(nb, ctx, c, g, pca, **kw)
    loss = tr.run(4)
    rl, rloss, _, _ = _oracle(port, c, g, pca, 4, **okw)
    assert np.array_equal(tr.layout(), rl)
    np.testing.assert_allclose(loss, rloss, rtol=1e-13, atol=0)


@pytest.mark.parametrize("head_only", [False, True])
def test_replay_star_graph_chains(port, ctx, head_only):
    """Every row of a cluster lists the cluster's first point (a star), so
    each worker's epoch is one long dependency chain through that point —
    the case the early neighbour forward and the position mailboxes exist
    for — plus repeats of the centre inside some lists: bit-identical."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    a = np.asarray(c.assignment)
    off = np.asarray(g.offsets).astype(np.int64)
    nbr = np.asarray(g.neighbors).copy()
    first = {int(r): int(np.flatnonzero(a == r)[0]) for r in np.unique(a)}
    for i in range(len(a)):
        ctr = first[int(a[i])]
        if ctr != i and off[i + 1] > off[i]:
            nbr[off[i]] = ctr                       # the centre leads every list
            if i % 7 == 0 and off[i + 1] - off[i] > 3:
                nbr[off[i] + 2] = ctr               # and repeats in some
    g2 = nb.KnnGraph(len(a), g.k, g.offsets, nbr, np.zeros(0))
    kw = dict(epochs=10, workers=4, seed=13, head_only=head_only)
    okw = dict(epochs=10, workers=4, seed=13, head_only=int(head_only))
    cfg = nb.TrainConfig(**kw)
    tr = nb.Trainer(g2, nb.ClusterAssignment(c.assignment, c.n_clusters, c.dims, c.centroids,
                                             c.sizes), pca, cfg, ctx=ctx)
    loss = tr.run(4)
    from oracle import train_config
    rl, rloss, _, _ = port.train_epochs(c.assignment, c.n_clusters, g.offsets, nbr, g.k,
                                        train_config(**okw), pca, 0, 4)
    assert np.array_equal(tr.layout(), rl)
    np.testing.assert_allclose(loss, rloss, rtol=1e-13, atol=0)


def test_replay_ragged_neighbor_lists(port, ctx):
    """Clusters smaller than k+1 give short lists (knn.hpp:77-83)."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(600, 8, 40, 40, 15)
    counts = np.diff(g.offsets)
    assert counts.min() < 15  # the case is actually ragged
    kw = dict(epochs=5, workers=4, seed=5)
    tr = _trainer(nb, ctx, c, g, pca, **kw)
    loss = tr.run(5)
    rl, rloss, _, _ = _oracle(port, c, g, pca, 5, **kw)
    assert np.array_equal(tr.layout(), rl)
    np.testing.assert_allclose(loss, rloss, rtol=1e-13, atol=0)


def test_divergence_error_matches_reference(port, ctx):
    """optimizer.hpp:215-227: a huge lr0 diverges; same kind and message."""
    import paper_2505_15511_b200 as nb
    from oracle import OracleError
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=10, workers=1, seed=7, lr0=1e14)
    tr = _trainer(nb, ctx, c, g, pca, **kw)
    with pytest.raises(nb.NomadError) as ei:
        tr.run(3)
    with pytest.raises(OracleError) as eo:
        _oracle(port, c, g, pca, 3, **kw)
    assert ei.value.kind == "Divergence" == eo.value.kind
    assert ei.value.message == eo.value.msg


def test_parameter_errors(ctx):
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    with pytest.raises(nb.NomadError) as e:
        _trainer(nb, ctx, c, g, pca, epochs=10, workers=9)
    assert e.value.kind == "Parameter"
    tr = _trainer(nb, ctx, c, g, pca, epochs=2, workers=1)
    tr.run(2)
    with pytest.raises(nb.NomadError) as e:
        tr.run(1)
    assert e.value.kind == "Parameter"


@pytest.mark.parametrize("workers,double_float", [(1, False), (4, False), (4, True)])
def test_hogwild_statistical_parity(port, ctx, workers, double_float):
    """Throughput mode (double-float or f64 position rows): same loss
    trajectory as the reference within 5%."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=30, workers=workers, seed=7)
    tr = _trainer(nb, ctx, c, g, pca, sgd_mode="hogwild", hogwild_double_float=double_float, **kw)
    loss = tr.run(30)
    lay = tr.layout()
    assert np.isfinite(lay).all()
    _, rloss, _, _ = _oracle(port, c, g, pca, 30, **kw)
    assert abs(loss[-5:].mean() - rloss[-5:].mean()) < 0.05 * rloss[-5:].mean()
    e, edges = tr.progress()
    assert e == 30 and edges == 30 * 3000 * 20


def test_config_a_replay(port, ctx):
    """BASELINE config A (20k x 64, k=15, single shard): 3 epochs bit-exact."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(20000, 64, 10, 5, 15)
    kw = dict(epochs=200, workers=1, seed=7)
    tr = _trainer(nb, ctx, c, g, pca, **kw)
    loss = tr.run(3)
    rl, rloss, _, _ = _oracle(port, c, g, pca, 3, **kw)
    assert np.array_equal(tr.layout(), rl)
    np.testing.assert_allclose(loss, rloss, rtol=1e-13, atol=0)


def _many_clusters(C, per, k, seed=3):
    """C clusters of `per` points (cluster of i = i mod C), lists of the other
    min(k, per - 1) members: more cells than the shared-memory tables hold."""
    n = C * per
    rng = np.random.default_rng(seed)
    i = np.arange(n)
    a = (i % C).astype(np.uint32)
    q = i // C
    m = min(k, per - 1)
    nb = np.stack([a + C * ((q + r) % per) for r in range(1, m + 1)], 1).astype(np.uint32)
    offsets = (np.arange(n + 1) * m).astype(np.uint32)
    return n, a, offsets, nb.reshape(-1), rng.normal(size=(n, 2))


@pytest.mark.parametrize("mode", ["replay", "hogwild"])
def test_many_clusters_global_cell_tables(port, ctx, mode):
    """C = 9000 > the old shared-memory cap (~8450 cells): the cell
    tables move to global memory. The reference's auto C = ceil(n / 4096)
    (optimizer.hpp:73-77) reaches 14.6k at 60M rows."""
    import paper_2505_15511_b200 as nb
    from oracle import train_config
    C = 9000
    n, a, off, nbr, init = _many_clusters(C, 6, 15)
    kw = dict(epochs=10, workers=8, seed=7)
    # 6-point clusters: the throughput kernel's concurrency is capped low
    # (<= 13 heads in flight per 6750-point shard) so that concurrent heads
    # rarely share a cluster and the trajectory is comparable
    tr = nb.Trainer(nb.KnnGraph(n, 15, off, nbr, np.zeros(0)),
                    nb.ClusterAssignment(a, C, 0, np.zeros(0), np.zeros(0)), init,
                    nb.TrainConfig(sgd_mode=mode, hogwild_cap=512, **kw), ctx=ctx)
    n_run = 2 if mode == "replay" else 6
    loss = tr.run(n_run)
    rl, rloss, rmeans, _ = port.train_epochs(a, C, off, nbr, 15, train_config(**kw), init, 0, n_run)
    if mode == "replay":
        assert np.array_equal(tr.layout(), rl)
        np.testing.assert_allclose(loss, rloss, rtol=1e-13, atol=0)
        assert np.array_equal(tr.means()[0], rmeans)
    else:
        assert np.isfinite(tr.layout()).all()
        assert abs(loss[-3:].mean() - rloss[-3:].mean()) < 0.05 * rloss[-3:].mean()
        assert tr.progress()[1] == n_run * n * (5 + 5)


def test_list_longer_than_k_is_rejected(ctx):
    """k_build_ell: a list longer than k or naming another
    worker's point is a Parameter error, not a silent out-of-table read."""
    import paper_2505_15511_b200 as nb
    n, a, off, nbr, init = _many_clusters(64, 20, 15)
    g = nb.KnnGraph(n, 12, off, nbr, np.zeros(0))  # lists hold 15 > k = 12
    with pytest.raises(nb.NomadError) as e:
        nb.Trainer(g, nb.ClusterAssignment(a, 64, 0, np.zeros(0), np.zeros(0)), init,
                   nb.TrainConfig(epochs=2, workers=2, k=12), ctx=ctx)
    assert e.value.kind == "Parameter"
    bad = nbr.copy().reshape(n, 15)
    bad[0, 0] = 1  # point 1 is in cluster 1; with W=64 workers it is another worker's
    with pytest.raises(nb.NomadError) as e:
        nb.Trainer(nb.KnnGraph(n, 15, off, bad.reshape(-1), np.zeros(0)),
                   nb.ClusterAssignment(a, 64, 0, np.zeros(0), np.zeros(0)), init,
                   nb.TrainConfig(epochs=2, workers=64), ctx=ctx)
    assert e.value.kind == "Parameter"


@pytest.mark.parametrize("mode", ["all_but_own", "head_only"])
@pytest.mark.parametrize("double_float", [False, True])
def test_hogwild_ablation_modes(port, ctx, mode, double_float):
    """The throughput kernel's ablation instances (k_sgd_hogwild<..., ABO>,
    head_only; optimizer.hpp:264-277, :294): loss trajectory within 5% of the
    reference's in the same mode, every edge counted."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=30, workers=4, seed=7)
    okw = dict(kw)
    if mode == "all_but_own":
        kw["approx"] = "non-own-cluster"
        okw["approx_all_but_own"] = 1
    else:
        kw["head_only"] = True
        okw["head_only"] = 1
    tr = _trainer(nb, ctx, c, g, pca, sgd_mode="hogwild", hogwild_double_float=double_float, **kw)
    loss = tr.run(30)
    assert np.isfinite(tr.layout()).all()
    _, rloss, _, _ = _oracle(port, c, g, pca, 30, **okw)
    assert abs(loss[-5:].mean() - rloss[-5:].mean()) < 0.05 * rloss[-5:].mean()
    assert tr.progress()[1] == 30 * 3000 * 20
