"""GPU quality metrics (metrics.hpp:113-243) bit-identical to the reference's
own metric code (oracle/_ref): NP@k (all rows and sampled, ties, k at the
filter-size boundary) and random-triplet accuracy."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def data(port):
    x = port.gaussian_mixture(3000, 24, 6, 10.0, 11)
    rng = np.random.default_rng(3)
    lay = rng.normal(size=(3000, 2)) * 5.0
    return x, lay


@pytest.mark.parametrize("k,sample,seed", [(10, 0, 0), (10, 500, 5), (1, 300, 2), (24, 400, 9),
                                           (25, 200, 1), (56, 100, 4), (57, 100, 6),
                                           (100, 200, 8), (300, 50, 3)])
def test_np_bit_exact(ref, ctx, data, k, sample, seed):
    import paper_2505_15511_b200 as nb
    x, lay = data
    v, se = nb.neighborhood_preservation(x, lay, k, sample, seed, ctx=ctx)
    rv, rse = ref.neighborhood_preservation(x, lay, k, sample=sample, seed=seed)
    assert v == rv and se == rse


def test_np_ties_and_odd_dims(ref, ctx, port):
    """Duplicated rows (ties at distance 0 in both spaces, decided by id) and a
    dimension that is not a multiple of 4 (scalar cp.async pieces)."""
    import paper_2505_15511_b200 as nb
    base = port.gaussian_mixture(300, 13, 3, 10.0, 2)
    x = np.ascontiguousarray(np.repeat(base, 4, axis=0))
    lay = np.repeat(np.random.default_rng(1).integers(0, 5, size=(300, 2)).astype(np.float64), 4, axis=0)
    for k, sample in [(5, 0), (15, 200)]:
        v, se = nb.neighborhood_preservation(x, lay, k, sample, 3, ctx=ctx)
        rv, rse = ref.neighborhood_preservation(x, lay, k, sample=sample, seed=3)
        assert v == rv and se == rse


@pytest.mark.parametrize("count,seed", [(1, 0), (5000, 3), (100000, 7)])
def test_triplet_bit_exact(ref, ctx, data, count, seed):
    import paper_2505_15511_b200 as nb
    x, lay = data
    v, se = nb.random_triplet_accuracy(x, lay, count, seed, ctx=ctx)
    rv, rse = ref.random_triplet_accuracy(x, lay, count, seed)
    assert v == rv and se == rse


def test_metric_errors(ctx, data):
    import paper_2505_15511_b200 as nb
    x, lay = data
    with pytest.raises(nb.NomadError):
        nb.neighborhood_preservation(x[:5], lay[:5], 5, ctx=ctx)  # k >= n
    with pytest.raises(nb.NomadError):
        nb.random_triplet_accuracy(x[:2], lay[:2], 10, ctx=ctx)  # n < 3
    with pytest.raises(nb.NomadError):
        nb.random_triplet_accuracy(x, lay, 0, ctx=ctx)


@pytest.mark.parametrize("k", [5, 10, 15])
def test_np_ann_bit_exact(ref, ctx, port, k):
    """NP-ann (graph neighbourhoods vs exact 2-D), incl. ragged lists and a
    singleton cluster (empty list)."""
    import paper_2505_15511_b200 as nb
    from common import index_case
    x, c, g, _ = index_case(3000, 32, 10, 8, 15)
    lay = np.random.default_rng(k).normal(size=(3000, 2))
    v = nb.neighborhood_preservation_ann(nb.KnnGraph(3000, 15, g.offsets, g.neighbors, g.distances),
                                         lay, k, ctx=ctx)
    assert v == ref.neighborhood_preservation_ann(g.offsets, g.neighbors, lay, k)
    off = np.concatenate([[0], np.cumsum(np.arange(300) % 4)]).astype(np.uint32)
    nbr = (np.arange(off[-1]) * 7 % 300).astype(np.uint32)
    lay2 = np.round(np.random.default_rng(1).normal(size=(300, 2)), 1)  # ties in 2-D
    v2 = nb.neighborhood_preservation_ann(nb.KnnGraph(300, 3, off, nbr, np.zeros(0)), lay2, k, ctx=ctx)
    assert v2 == ref.neighborhood_preservation_ann(off, nbr, lay2, k)
