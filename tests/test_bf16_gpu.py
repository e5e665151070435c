"""bf16 datasets (the 60M x 768 bf16 configuration's storage) on the B200.

bf16 values widen exactly to f32, so every index-build result on a bf16
dataset must equal the reference's result on the widened f32 data: LSH
seeding, k-means and the tolerance bit-identical to the oracle; the bf16-mode
kNN graph and recall, PCA (exact and fast), NP@k, triplet accuracy and fit()
identical to the f32 call on the widened rows. Also: the
grouped tensor-core copy (clusters processed in memory-bounded groups) equals
the single-group result, and the exact kNN modes on bf16 rows equal the exact
f32 build on the widened rows."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bf16_pair(nb, ctx, n, d, blobs, seed=42):
    import torch
    x16 = nb.generate_mixture(n, d, blobs, 10.0, seed, ctx=ctx, dtype="bf16")
    return x16, x16.float()


def test_generator_bf16_is_rounded_f32(ctx):
    import torch
    import paper_2505_15511_b200 as nb
    x32 = nb.generate_mixture(5000, 96, 7, 10.0, 3, ctx=ctx)
    x16 = nb.generate_mixture(5000, 96, 7, 10.0, 3, ctx=ctx, dtype="bf16")
    assert x16.dtype == torch.bfloat16
    assert torch.equal(x16.view(torch.int16), x32.to(torch.bfloat16).view(torch.int16))


@pytest.mark.parametrize("n,d,blobs,C,seed", [(3000, 32, 10, 8, 7), (2000, 48, 3, 40, 11)])
def test_lsh_kmeans_bf16_vs_oracle(port, ctx, n, d, blobs, C, seed):
    import paper_2505_15511_b200 as nb
    x16, xw = _bf16_pair(nb, ctx, n, d, blobs, 40 + seed)
    xh = xw.cpu().numpy()
    r0 = port.lsh_init(xh, C, seed)
    g0 = nb.lsh_init(x16, C, seed, ctx=ctx)
    assert np.array_equal(g0.assignment, r0.assignment)
    assert np.array_equal(g0.centroids, r0.centroids)
    tol = port.default_kmeans_tol(xh)
    assert nb.default_kmeans_tol(x16, ctx=ctx) == tol
    r1 = port.kmeans_em(xh, r0, 100, tol)
    g1 = nb.kmeans_em(x16, g0, 100, tol, ctx=ctx)
    assert np.array_equal(g1.assignment, r1.assignment)
    assert np.array_equal(g1.centroids, r1.centroids)
    g2 = nb.kmeans_em_default_tol(x16, g0, 100, ctx=ctx)
    assert np.array_equal(g2.assignment, r1.assignment)


@pytest.mark.parametrize("n,d,blobs,C", [(20000, 128, 12, 6), (6000, 768, 8, 3)])
def test_knn_bf16_dataset_equals_widened(ctx, n, d, blobs, C):
    import paper_2505_15511_b200 as nb
    x16, xw = _bf16_pair(nb, ctx, n, d, blobs)
    c = nb.kmeans_em_default_tol(x16, nb.lsh_init(x16, C, 7, ctx=ctx), 100, ctx=ctx)
    cw = nb.kmeans_em_default_tol(xw, nb.lsh_init(xw, C, 7, ctx=ctx), 100, ctx=ctx)
    assert np.array_equal(c.assignment, cw.assignment)
    g16 = nb.build_knn(x16, c, 15, mode="bf16", ctx=ctx)
    gw = nb.build_knn(xw, c, 15, mode="bf16", ctx=ctx)
    assert np.array_equal(g16.offsets, gw.offsets)
    assert np.array_equal(g16.neighbors, gw.neighbors)
    assert np.array_equal(g16.distances, gw.distances)
    r16 = nb.knn_recall(x16, c, g16, sample=500, seed=3, ctx=ctx)
    rw = nb.knn_recall(xw, c, gw, sample=500, seed=3, ctx=ctx)
    assert r16 == rw and r16 > 0.99


@pytest.mark.parametrize("mode", ["bf16", "exact"])
def test_knn_grouped_copy_equals_single(ctx, mode, monkeypatch):
    """Force the tensor-core stage to build its 16-bit copy in several
    memory-bounded cluster groups; the graph must not change."""
    import paper_2505_15511_b200 as nb
    x = nb.generate_mixture(12000, 64, 9, 10.0, 5, ctx=ctx)
    c = nb.kmeans_em_default_tol(x, nb.lsh_init(x, 9, 7, ctx=ctx), 100, ctx=ctx)
    g1 = nb.build_knn(x, c, 15, mode=mode, ctx=ctx)
    monkeypatch.setenv("NOMAD_B200_TC_ROW_BUDGET", "2000")
    g2 = nb.build_knn(x, c, 15, mode=mode, ctx=ctx)
    assert np.array_equal(g1.offsets, g2.offsets)
    assert np.array_equal(g1.neighbors, g2.neighbors)
    assert np.array_equal(g1.distances, g2.distances)


def test_pca_and_triplets_bf16_equal_widened(ctx):
    import paper_2505_15511_b200 as nb
    x16, xw = _bf16_pair(nb, ctx, 4000, 48, 6)
    for fast in (False, True):
        a = nb.pca_init(x16, 7, ctx=ctx, fast=fast)
        b = nb.pca_init(xw, 7, ctx=ctx, fast=fast)
        assert np.array_equal(a, b)
    lay = nb.pca_init(xw, 7, ctx=ctx)
    assert (nb.random_triplet_accuracy(x16, lay, 20000, 3, ctx=ctx)
            == nb.random_triplet_accuracy(xw, lay, 20000, 3, ctx=ctx))


@pytest.mark.parametrize("n,d,k", [(6000, 48, 10), (40000, 64, 30)])
def test_neighborhood_preservation_bf16_equals_widened(ctx, n, d, k):
    """NP@k on bf16 rows: the global high-d search widens the rows chunk by
    chunk for the FFMA filter (many candidate partitions); same value and
    standard error as on the widened f32 rows."""
    import paper_2505_15511_b200 as nb
    x16, xw = _bf16_pair(nb, ctx, n, d, 9)
    lay = nb.pca_init(xw, 7, ctx=ctx)
    assert (nb.neighborhood_preservation(x16, lay, k, 300, 1, ctx=ctx)
            == nb.neighborhood_preservation(xw, lay, k, 300, 1, ctx=ctx))


@pytest.mark.parametrize("mode", ["exact", "exact_ffma"])
@pytest.mark.parametrize("n,d,blobs,C", [(8000, 64, 6, 6), (20000, 64, 24, 4), (3000, 768, 5, 2)])
def test_knn_exact_modes_bf16_equal_widened(ctx, mode, n, d, blobs, C):
    """Exact kNN on bf16 rows (tensor-core certificate, sub-cluster stage and
    the FFMA filter on per-cluster widened copies, exhaustive fallback): ids
    and fp64 distances identical to the exact build on the widened f32 rows
    (which tests/test_knn_gpu.py pins to the reference)."""
    import paper_2505_15511_b200 as nb
    x16, xw = _bf16_pair(nb, ctx, n, d, blobs)
    c = nb.kmeans_em_default_tol(xw, nb.lsh_init(xw, C, 7, ctx=ctx), 100, ctx=ctx)
    g16 = nb.build_knn(x16, c, 15, mode=mode, ctx=ctx)
    gw = nb.build_knn(xw, c, 15, mode=mode, ctx=ctx)
    assert np.array_equal(g16.offsets, gw.offsets)
    assert np.array_equal(g16.neighbors, gw.neighbors)
    assert np.array_equal(g16.distances, gw.distances)


def test_fit_bf16_rows_equals_widened(ctx):
    """fit() end to end on bf16 rows (bf16 kNN mode, GPU PCA, replay epochs)
    is bit-identical to fit() on the widened f32 rows."""
    import paper_2505_15511_b200 as nb
    x16, xw = _bf16_pair(nb, ctx, 3000, 32, 6)
    cfg = nb.TrainConfig(epochs=3, workers=2, seed=7, knn_mode="bf16", n_clusters=4)
    a = nb.fit(x16, cfg, ctx=ctx)
    b = nb.fit(xw, cfg, ctx=ctx)
    assert np.array_equal(a, b)
