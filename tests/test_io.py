"""Data I/O at the path's ends (dataset.hpp:122-173, :223-250) against the
reference library (oracle/_ref): the layout CSV is byte-identical, the raw-f32
loader returns the same values and fails with the same kind and message.
Host-only entry points: these run without a GPU."""
import os

import numpy as np
import pytest

import paper_2505_15511_b200 as nb
from oracle import OracleError


def _lay(n, seed=0):
    r = np.random.default_rng(seed)
    lay = r.normal(size=(n, 2)) * 10.0 ** r.integers(-12, 12, size=(n, 2))
    if n >= 2:
        lay[0] = [0.0, -0.0]
        lay[1] = [1.0 / 3.0, -2.0 ** -1074]
    return lay


@pytest.mark.parametrize("n,with_ids,with_labels", [(0, False, False), (1, False, False),
                                                    (5000, False, False), (300, True, True),
                                                    (140000, False, True)])
def test_layout_csv_byte_identical(ref, tmp_path, n, with_ids, with_labels):
    lay = _lay(n)
    ids = [f"p{i}" for i in range(n)] if with_ids else None
    labels = [f"c{i % 7}" for i in range(n)] if with_labels else None
    a, b = str(tmp_path / "ours.csv"), str(tmp_path / "ref.csv")
    nb.save_layout(lay, a, ids, labels)
    ref.save_layout(lay, b, ids, labels)
    assert open(a, "rb").read() == open(b, "rb").read()


def test_layout_f64_round_trip(tmp_path):
    lay = _lay(1000, 3)
    p = str(tmp_path / "l.f64")
    nb.save_layout_f64(lay, p)
    assert np.array_equal(np.fromfile(p, np.float64).reshape(-1, 2), lay)


def _raw(tmp_path, arr, name="x.f32"):
    p = str(tmp_path / name)
    np.ascontiguousarray(arr, "<f4").tofile(p)
    return p


@pytest.mark.parametrize("rows,dims", [(50, 7), (50, 0), (0, 7)])
def test_load_raw_matches_reference(ref, tmp_path, rows, dims):
    x = np.random.default_rng(1).normal(size=(50, 7)).astype(np.float32)
    p = _raw(tmp_path, x)
    ours = nb.load_vectors_raw(p, rows, dims)
    theirs = ref.load_vectors_raw(p, rows, dims)
    assert ours.shape == theirs.shape == (50, 7)
    assert np.array_equal(ours.view(np.uint32), theirs.view(np.uint32))


def _same_error(fn_ours, fn_ref):
    with pytest.raises(nb.NomadError) as eo:
        fn_ours()
    with pytest.raises(OracleError) as er:
        fn_ref()
    assert eo.value.kind == er.value.kind
    assert eo.value.message == er.value.msg


def test_load_raw_errors_match_reference(ref, tmp_path):
    x = np.arange(42, dtype=np.float32).reshape(6, 7)
    p = _raw(tmp_path, x)
    for rows, dims in [(0, 0), (5, 7), (4, 0), (0, 5), (6, 8)]:
        _same_error(lambda: nb.load_vectors_raw(p, rows, dims),
                    lambda: ref.load_vectors_raw(p, rows, dims))
    odd = str(tmp_path / "odd.f32")
    open(odd, "wb").write(b"\0" * 10)
    _same_error(lambda: nb.load_vectors_raw(odd, 0, 1), lambda: ref.load_vectors_raw(odd, 0, 1))
    bad = x.copy()
    bad[3, 5] = np.nan
    bad[4, 0] = np.inf
    pb = _raw(tmp_path, bad, "bad.f32")
    _same_error(lambda: nb.load_vectors_raw(pb, 6, 7), lambda: ref.load_vectors_raw(pb, 6, 7))
    one = _raw(tmp_path, x[:1], "one.f32")
    _same_error(lambda: nb.load_vectors_raw(one, 1, 7), lambda: ref.load_vectors_raw(one, 1, 7))
    missing = str(tmp_path / "nope.f32")
    _same_error(lambda: nb.load_vectors_raw(missing, 1, 1),
                lambda: ref.load_vectors_raw(missing, 1, 1))
