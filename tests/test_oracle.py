"""CPU: the C restatement (oracle/nomad_oracle.c) is pinned (1) to golden
fixtures generated from the reference itself (tests/make_golden.py ->
tests/golden/reference_goldens.json) and (2) directly to the compiled
reference (oracle/_ref) where present; plus SPEC.md known answers."""
import json
import os

import numpy as np
import pytest

from common import sha

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_goldens.json")))


def test_rng_known_answers(port):
    r = G["rng"]
    assert hex(port.stream_seed(0, 0)) == r["stream_seed_0_0"]
    assert [hex(int(v)) for v in port.rng_u64(5, 8)] == r["mt_u64_seed5_first8"]
    assert sha(port.rng_gaussian(5, 1001)) == r["gaussian_seed5_sha_1001"]
    assert sha(port.rng_uniform_index(5, 77, 1000)) == r["uniform_index_seed5_b77_sha_1000"]
    assert [float(v).hex() for v in port.inverse_rank_weights(15)] == r["inverse_rank_weights_15"]
    assert port.lr_schedule(9, 10, 100.0).hex() == r["lr_9_of_10_lr0_100"]


def test_spec_known_answers(port):
    # rng.hpp:25-30 splitmix64(0)
    from oracle import Oracle
    lib = port.lib
    lib.orc_mix_seed.restype = __import__("ctypes").c_uint64
    lib.orc_mix_seed.argtypes = [__import__("ctypes").c_uint64]
    assert lib.orc_mix_seed(0) == 0xE220A8397B1DCDAF
    # SPEC.md:195 inverse_rank_weights(2)
    w = port.inverse_rank_weights(2)
    assert w[0] == 0.62245933120185448 and w[1] == 0.37754066879814541
    w15 = port.inverse_rank_weights(15)
    assert w15[0] == 0.1403794162597248 and w15[14] == 0.055202902845087214
    # SPEC.md:385 lr at epoch 9/10 (oracle bits, not the math)
    assert port.lr_schedule(9, 10, 100.0) == 9.9999999999999982
    # SPEC.md:394 LPT sizes {5,3,3,3}, W=2 -> {5,3} vs {3,3}
    a = np.array([0] * 5 + [1] * 3 + [2] * 3 + [3] * 3, np.uint32)
    c2w, pts = port.shard_clusters(a, 4, 2)
    assert c2w.tolist() == [0, 1, 1, 0]
    # SPEC.md:138 collinear 0,1,3 one cluster k=1
    x = np.array([[0.0], [1.0], [3.0]], np.float32)
    from oracle import Clusters
    cl = Clusters(np.zeros(3, np.uint32), np.zeros(1), np.array([3], np.uint32), 1, 1)
    g = port.build_knn(x, cl, 1)
    assert g.neighbors.tolist() == [1, 0, 1] and g.distances.tolist() == [1.0, 1.0, 4.0]
    # SPEC.md:402 gather_means: (0,0),(2,2) -> (1,1)
    m = port.gather_means(np.array([[0.0, 0.0], [2.0, 2.0]]), np.zeros(2, np.uint32), 1)
    assert m.tolist() == [[1.0, 1.0]]


@pytest.mark.parametrize("case", ["small_w4", "ragged_w4", "config_a_w1", "config_a_w4"])
def test_port_matches_reference_goldens(port, case):
    from oracle import train_config
    gc = G["cases"][case]
    n, d, blobs, ncl, k, W, nrun, sched = gc["shape"]
    if n > 5000 and os.environ.get("NOMAD_FAST_TESTS"):
        pytest.skip("large golden case skipped (NOMAD_FAST_TESTS)")
    x = port.gaussian_mixture(n, d, blobs, 10.0, 42)
    assert sha(x) == gc["data"]
    c0 = port.lsh_init(x, ncl, 7)
    assert sha(c0.assignment) == gc["lsh_assignment"] and sha(c0.centroids) == gc["lsh_centroids"]
    tol = port.default_kmeans_tol(x)
    assert tol.hex() == gc["default_kmeans_tol"]
    c, qe = port.kmeans_em(x, c0, 100, tol, trace=True)
    assert sha(c.assignment) == gc["km_assignment"] and sha(c.centroids) == gc["km_centroids"]
    assert [float(v).hex() for v in qe] == gc["qe_trace"]
    g = port.build_knn(x, c, k)
    assert sha(g.offsets) == gc["knn_offsets"]
    assert sha(g.neighbors) == gc["knn_neighbors"] and sha(g.distances) == gc["knn_distances"]
    pca = port.pca_init(x, 7)
    assert sha(pca) == gc["pca"]
    lay, loss, means, _ = port.train_epochs(c.assignment, ncl, g.offsets, g.neighbors, k,
                                            train_config(epochs=sched, workers=W, seed=7), pca,
                                            0, nrun)
    assert sha(lay) == gc["layout"]
    assert [float(v).hex() for v in loss] == gc["epoch_loss"]
    assert sha(means) == gc["final_means"]


def test_port_matches_reference_fit_and_modes(port, ref):
    """Direct oracle-vs-reference on a fresh seed: whole fit() and the ablation
    modes of the epoch loop (optimizer.hpp:264-277, :294)."""
    from oracle import train_config
    x = port.gaussian_mixture(1500, 12, 6, 10.0, 99)
    cfg = train_config(epochs=6, workers=3, seed=5, n_clusters=6)
    f = ref.fit(x, cfg)
    c = port.lsh_init(x, 6, 5)
    c = port.kmeans_em(x, c, 100, port.default_kmeans_tol(x))
    assert np.array_equal(c.assignment, f["assignment"])
    g = port.build_knn(x, c, 15)
    assert np.array_equal(g.neighbors, f["neighbors"]) and np.array_equal(g.distances, f["distances"])
    pca = port.pca_init(x, 5)
    assert np.array_equal(pca, f["pca"])
    lay, loss, means, _ = port.train_epochs(c.assignment, 6, g.offsets, g.neighbors, 15, cfg, pca)
    assert np.array_equal(lay, f["layout"]) and np.array_equal(loss, f["epoch_loss"])
    assert np.array_equal(means, f["final_means"])
    for extra in (dict(approx_all_but_own=1), dict(head_only=1)):
        cfg2 = train_config(epochs=6, workers=3, seed=5, **extra)
        a = port.train_epochs(c.assignment, 6, g.offsets, g.neighbors, 15, cfg2, pca)
        b = ref.train_epochs(c.assignment, 6, g.offsets, g.neighbors, 15, cfg2, pca)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_gradient_matches_reference_and_finite_differences(port, ref):
    """objective.hpp:178-237 analytic gradient: port == reference bit-exact, and
    the head gradient agrees with central finite differences of the loss
    (SPEC.md acceptance #4)."""
    rng = np.random.default_rng(0)
    lay = rng.normal(size=(40, 2))
    nb = np.arange(1, 16, dtype=np.uint32)
    w = port.inverse_rank_weights(15)
    negs = np.array([20, 21, 22, 23, 0], np.uint32)
    means = rng.normal(size=(6, 2)) * 3
    remote = np.array([1, 3, 4], np.uint32)
    probs = np.array([0.1, 0.2, 0.15])
    a = port.nomad_gradient(lay, 0, nb, w, negs, remote, probs, means, 0.55, 5)
    b = ref.nomad_gradient(lay, 0, nb, w, negs, remote, probs, means, 0.55, 5)
    assert a[0] == b[0] and np.array_equal(a[1], b[1])
    # finite differences on the head (negatives' positions enter via bg only)
    negs2 = np.array([20, 21, 22, 23, 24], np.uint32)
    loss0, g = port.nomad_gradient(lay, 0, nb, w, negs2, remote, probs, means, 0.55, 5)
    for dim in range(2):
        h = 1e-6
        lp, lm = lay.copy(), lay.copy()
        lp[0, dim] += h
        lm[0, dim] -= h
        fp = port.nomad_gradient(lp, 0, nb, w, negs2, remote, probs, means, 0.55, 5)[0]
        fm = port.nomad_gradient(lm, 0, nb, w, negs2, remote, probs, means, 0.55, 5)[0]
        assert abs((fp - fm) / (2 * h) - g[0, dim]) < 1e-5 * max(1.0, abs(g[0, dim]))


def test_oracle_error_kinds(port):
    from oracle import OracleError
    x = port.gaussian_mixture(50, 4, 2, 10.0, 1)
    with pytest.raises(OracleError) as e:
        port.lsh_init(x, 1, 0)
    assert e.value.kind == "Parameter" and "cluster count must be in [2, n]" in e.value.msg
    with pytest.raises(OracleError) as e:
        port.pca_init(np.ones((10, 3), np.float32))
    assert e.value.kind == "Degenerate"


@pytest.mark.parametrize("which", ["port", "reference"])
def test_row_checkers_match_whole_builds(which):
    """The per-row checkers used at configs B/C (knn_rows, nearest_centroid_rows,
    cluster_centroid) reproduce the whole reference build on a small case."""
    from oracle import Oracle, available
    if not available(which):
        pytest.skip(f"{which} checker not built")
    o = Oracle(which)
    x = Oracle("port").gaussian_mixture(3000, 16, 5, 10.0, 42)
    c = o.lsh_init(x, 4, 7)
    c = o.kmeans_em(x, c, 100, o.default_kmeans_tol(x))
    g = o.build_knn(x, c, 15)
    for r in range(4):
        mem = np.nonzero(c.assignment == r)[0]
        q = np.arange(0, len(mem), 29)
        ids, ds = o.knn_rows(x[mem], mem, q, 15)
        for t, qi in enumerate(q):
            i = mem[qi]
            assert np.array_equal(ids[t], g.neighbors[g.offsets[i]:g.offsets[i + 1]])
            assert np.array_equal(ds[t], g.distances[g.offsets[i]:g.offsets[i + 1]])
        assert np.array_equal(o.cluster_centroid(x[mem]), c.centroids[r * 16:(r + 1) * 16])
    assert np.array_equal(o.nearest_centroid_rows(x, c.centroids), c.assignment)
