"""Device-side data I/O: the raw-f32 loader streaming into device memory
(dataset.hpp:122-173, GPU finiteness scan) and fit() checkpoints
(optimizer.hpp:463-469: `<prefix>.epoch<N>.csv` every N epochs)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_load_raw_to_device(ref, ctx, tmp_path):
    import paper_2505_15511_b200 as nb
    x = np.random.default_rng(2).normal(size=(20000, 300)).astype(np.float32)  # > 1 chunk
    p = str(tmp_path / "x.f32")
    x.tofile(p)
    t = nb.load_vectors_raw(p, 0, 300, device=True, ctx=ctx)
    assert t.is_cuda and tuple(t.shape) == (20000, 300)
    assert np.array_equal(t.cpu().numpy().view(np.uint32), x.view(np.uint32))
    x[12345, 17] = np.inf
    x[19999, 0] = np.nan
    x.tofile(p)
    with pytest.raises(nb.NomadError) as e:
        nb.load_vectors_raw(p, 20000, 300, device=True, ctx=ctx)
    from oracle import OracleError
    with pytest.raises(OracleError) as r:
        ref.load_vectors_raw(p, 20000, 300)
    assert e.value.kind == r.value.kind == "Validation"
    assert e.value.message == r.value.msg


def test_fit_checkpoints(port, ctx, tmp_path):
    import paper_2505_15511_b200 as nb
    x = port.gaussian_mixture(1500, 16, 4, 10.0, 3)
    prefix = str(tmp_path / "run")
    cfg = nb.TrainConfig(epochs=5, workers=2, n_clusters=4, seed=3, checkpoint_every=2,
                         checkpoint_prefix=prefix)
    y = nb.fit(x, cfg, ctx=ctx)
    assert sorted(os.listdir(tmp_path)) == ["run.epoch2.csv", "run.epoch4.csv"]
    # epoch-4 checkpoint = the replay trajectory after 4 of the 5 epochs
    cfg4 = nb.TrainConfig(epochs=5, workers=2, n_clusters=4, seed=3)
    c = nb.kmeans_em_default_tol(x, nb.lsh_init(x, 4, 3, ctx=ctx), 100, ctx=ctx)
    g = nb.build_knn(x, c, 15, ctx=ctx)
    tr = nb.Trainer(g, c, nb.pca_init(x, 3, ctx=ctx), cfg4, ctx=ctx)
    tr.run(4)
    ref_csv = str(tmp_path / "direct.csv")
    nb.save_layout(tr.layout(), ref_csv)
    tr.run(1)
    assert np.array_equal(tr.layout(), y)
    tr.close()
    assert open(prefix + ".epoch4.csv", "rb").read() == open(ref_csv, "rb").read()


@pytest.mark.parametrize("mode", ["replay", "hogwild"])
def test_resume_from_checkpoint(port, ctx, tmp_path, mode):
    """fit()-style checkpoint after 3 of 6 epochs, reloaded from the CSV into a
    fresh trainer + seek(3): replay mode continues bit-identically; hogwild
    continues the same schedule (epoch-keyed draws) to a comparable loss."""
    import paper_2505_15511_b200 as nb
    x = port.gaussian_mixture(3000, 16, 5, 10.0, 4)
    c = nb.kmeans_em_default_tol(x, nb.lsh_init(x, 6, 2, ctx=ctx), 100, ctx=ctx)
    g = nb.build_knn(x, c, 15, ctx=ctx)
    init = nb.pca_init(x, 2, ctx=ctx)
    cfg = nb.TrainConfig(epochs=6, workers=2, seed=2, sgd_mode=mode)
    full = nb.Trainer(g, c, init, cfg, ctx=ctx)
    l_full = full.run(6)
    y_full = full.layout()
    full.close()
    a = nb.Trainer(g, c, init, cfg, ctx=ctx)
    a.run(3)
    p = str(tmp_path / "ck.epoch3.csv")
    nb.save_layout(a.layout(), p)
    a.close()
    ck = np.loadtxt(p, delimiter=",", skiprows=1)[:, 1:3]
    b = nb.Trainer(g, c, ck, cfg, ctx=ctx)
    b.seek(3)
    l_res = b.run(3)
    y_res = b.layout()
    assert b.progress()[0] == 6
    b.close()
    if mode == "replay":
        assert np.array_equal(y_res, y_full)
        assert np.array_equal(np.asarray(l_res), np.asarray(l_full)[3:])
    else:
        assert abs(l_res[-1] - l_full[-1]) < 0.05 * abs(l_full[-1])


def test_staged_host_copies_roundtrip(ctx):
    """Bulk copies to / from pageable host memory go through the context's
    pinned two-buffer ring (hostcopy.cu, 64 MB chunks, several host threads):
    a layout of 5,000,003 rows (80 MB: two chunks, the second partial) set
    from and read back into fresh numpy arrays is unchanged, and equals the
    device-side read."""
    import torch
    import paper_2505_15511_b200 as nb
    n, C, k = 5_000_003, 8, 4
    rng = np.random.default_rng(5)
    a = (np.arange(n) % C).astype(np.uint32)
    q = np.arange(n) // C
    m = (n - a.astype(np.int64) + C - 1) // C
    nbr = np.stack([(a + C * ((q + t + 1) % m)).astype(np.uint32) for t in range(k)], 1).reshape(-1)
    off = (np.arange(n + 1, dtype=np.uint64) * k).astype(np.uint32)
    g = nb.KnnGraph(n, k, off, nbr, np.zeros(0))
    c = nb.ClusterAssignment(a, C, 16, np.zeros(0), np.zeros(0))
    init = rng.standard_normal((n, 2))
    tr = nb.Trainer(g, c, init, nb.TrainConfig(epochs=10, workers=2, seed=3, k=k), ctx=ctx)
    lay = tr.layout()
    assert np.array_equal(lay, init)
    new = rng.standard_normal((n, 2))
    tr.set_layout(new)
    dev = torch.empty((n, 2), dtype=torch.float64, device="cuda")
    tr.layout(dev)
    assert np.array_equal(dev.cpu().numpy(), new)
    assert np.array_equal(tr.layout(), new)


def test_host_dataset_upload_matches_device(ctx):
    """A host (pageable) dataset above the staging threshold gives the same
    k-means and kNN graph as the same rows already on the device."""
    import torch
    import paper_2505_15511_b200 as nb
    x = nb.generate_mixture(200_003, 64, 6, 10.0, 9, ctx=ctx)  # 51 MB of f32 rows
    xh = x.cpu().numpy()
    cd = nb.kmeans_em_default_tol(x, nb.lsh_init(x, 6, 7, ctx=ctx), 100, ctx=ctx)
    ch = nb.kmeans_em_default_tol(xh, nb.lsh_init(xh, 6, 7, ctx=ctx), 100, ctx=ctx)
    assert np.array_equal(cd.assignment, ch.assignment)
    assert np.array_equal(cd.centroids, ch.centroids)
    gd = nb.build_knn(x, cd, 15, ctx=ctx)
    gh = nb.build_knn(xh, ch, 15, ctx=ctx)
    assert np.array_equal(gd.offsets, gh.offsets)
    assert np.array_equal(gd.neighbors, gh.neighbors)
    assert np.array_equal(gd.distances, gh.distances)
    torch.cuda.synchronize()
