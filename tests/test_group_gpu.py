"""Multi-rank execution on one B200: a group of G ranks in one
process (nomad_b200_group_create) with the loopback exchange runs the same
code path per rank as G processes over NCCL — only the all-gather transport
differs. With W logical workers fixed, replay mode must be bit-identical to
the oracle (the reference's run_worker_epoch + gather_means, optimizer.hpp:
232-307, :411-442) for every G; hogwild mode must apply every edge update."""
import numpy as np
import pytest

from common import index_case

pytestmark = pytest.mark.gpu


def _views(nb, c, g):
    return (nb.KnnGraph(len(c.assignment), g.k, g.offsets, g.neighbors, g.distances),
            nb.ClusterAssignment(c.assignment, c.n_clusters, c.dims, c.centroids, c.sizes))


def _oracle(port, c, g, pca, n_run, **kw):
    from oracle import train_config
    return port.train_epochs(c.assignment, c.n_clusters, g.offsets, g.neighbors, g.k,
                             train_config(**kw), pca, 0, n_run)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_group_replay_bit_exact_for_every_rank_count(port, G):
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=10, workers=8, seed=7)
    grp = nb.Group([0] * G)
    assert grp.size == G and grp.loopback == (G > 1)
    gv, cv = _views(nb, c, g)
    tr = nb.Trainer(gv, cv, pca, nb.TrainConfig(**kw), group=grp)
    assert tr.ranks == G
    loss = tr.run(4)
    lay = tr.layout()
    rl, rloss, rmeans, _ = _oracle(port, c, g, pca, 4, **kw)
    assert np.array_equal(lay, rl), f"G={G}: layout differs from the oracle"
    np.testing.assert_allclose(loss, rloss, rtol=1e-13, atol=0)
    m, counts = tr.means()
    assert np.array_equal(m, rmeans)
    log = tr.comm_log()
    assert (log.epochs, log.messages) == (4, 4 * 8)
    e, edges = tr.progress()
    assert e == 4 and edges == 4 * 3000 * 20
    tr.close()
    grp.close()


def test_group_replay_set_layout_and_resume(port):
    """set_layout + seek on a 4-rank group equals an uninterrupted run."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=6, workers=8, seed=5)
    gv, cv = _views(nb, c, g)
    grp = nb.Group([0] * 4)
    a = nb.Trainer(gv, cv, pca, nb.TrainConfig(**kw), group=grp)
    a.run(2)
    mid = a.layout()
    b = nb.Trainer(gv, cv, pca, nb.TrainConfig(**kw), group=grp)
    b.set_layout(mid)
    b.seek(2)
    b.run(3)
    a.run(3)
    assert np.array_equal(a.layout(), b.layout())
    rl, _, _, _ = _oracle(port, c, g, pca, 5, **kw)
    assert np.array_equal(a.layout(), rl)


def test_group_hogwild_two_ranks(port):
    """G=2, W=8 throughput mode: every edge update lands, loss tracks the
    reference's trajectory within 5%."""
    import paper_2505_15511_b200 as nb
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=30, workers=8, seed=7)
    gv, cv = _views(nb, c, g)
    grp = nb.Group([0, 0])
    tr = nb.Trainer(gv, cv, pca, nb.TrainConfig(sgd_mode="hogwild", **kw), group=grp)
    loss = tr.run(30)
    lay = tr.layout()
    assert np.isfinite(lay).all()
    e, edges = tr.progress()
    assert e == 30 and edges == 30 * 3000 * 20
    _, rloss, _, _ = _oracle(port, c, g, pca, 30, **kw)
    assert abs(loss[-5:].mean() - rloss[-5:].mean()) < 0.05 * rloss[-5:].mean()
    m, _ = tr.means()
    assert np.isfinite(m).all()


def test_group_divergence_same_error_on_every_rank(port):
    """optimizer.hpp:215-227 through a 2-rank group: same kind and message as
    the reference; the ranks agree on one decision."""
    import paper_2505_15511_b200 as nb
    from oracle import OracleError
    x, c, g, pca = index_case(3000, 32, 10, 8, 15)
    kw = dict(epochs=10, workers=2, seed=7, lr0=1e14)
    gv, cv = _views(nb, c, g)
    grp = nb.Group([0, 0])
    tr = nb.Trainer(gv, cv, pca, nb.TrainConfig(**kw), group=grp)
    with pytest.raises(nb.NomadError) as ei:
        tr.run(3)
    with pytest.raises(OracleError) as eo:
        _oracle(port, c, g, pca, 3, **kw)
    assert ei.value.kind == "Divergence" == eo.value.kind
    assert ei.value.message == eo.value.msg


def test_group_rejects_mixed_device_lists():
    import paper_2505_15511_b200 as nb
    with pytest.raises(nb.NomadError) as e:
        nb.Group([0, 0, 1])
    assert e.value.kind == "Parameter"
