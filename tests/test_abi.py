"""CPU: the C-ABI library loads and exports every symbol include/nomad_b200.h
declares (no compute calls without a GPU); the Python mirror binds them all;
the product never imports the oracle; the C++ shim compiles."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "nomad_b200.h")).read()
    return sorted(set(re.findall(r"\b(nomad_b200_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2505_15511_b200 as nb
    path = nb._native.LIB_PATH
    assert os.path.exists(path), "run __graft_entry__.build() first"
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (nomad_b200_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = nb.lib()
    for s in declared_symbols():
        assert hasattr(lib, s)
    assert set(nb.EXPORTED) <= set(declared_symbols())


def test_library_is_sm100a_only():
    import paper_2505_15511_b200 as nb
    out = subprocess.run(["cuobjdump", "--list-elf", nb._native.LIB_PATH], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_default_config_matches_reference_defaults():
    import ctypes as C
    import paper_2505_15511_b200 as nb
    c = nb._native.TrainConfigC()
    nb.lib().nomad_b200_default_config(C.byref(c))
    py = nb.TrainConfig()
    # optimizer.hpp:45-61
    assert (c.epochs, c.k, c.negatives, c.local_draws, c.batch_size, c.workers, c.n_clusters,
            c.seed, c.lr0, c.kmeans_max_iters, c.kmeans_tol) == \
        (200, 15, 5, 5, 1024, 1, 0, 0, 0.0, 100, -1.0)
    assert (py.epochs, py.k, py.negatives, py.local_draws, py.batch_size) == (200, 15, 5, 5, 1024)


def test_no_device_means_loud_error():
    """Without a GPU the context refuses to be created (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2505_15511_b200 as nb
    with pytest.raises(nb.NomadError) as e:
        nb.Context(0)
    assert e.value.kind == "Internal"


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2505_15511_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("Oracle", ""), f


def test_config_mirror():
    import paper_2505_15511_b200 as nb
    cfg = nb.TrainConfig(workers=4)
    assert cfg.resolve_clusters(20000) == 5      # optimizer.hpp:73-77
    assert cfg.resolve_clusters(3) == 3
    assert cfg.resolve_lr0(20000) == 2000.0      # optimizer.hpp:79-81
    with pytest.raises(nb.NomadError):
        nb.TrainConfig(workers=0).validate()
    with pytest.raises(nb.NomadError):
        nb.TrainConfig(workers=4, n_clusters=2).validate()


def test_dataset_view_dtype_plumbing():
    """The dataset view carries dtype (appended field, 0 = f32): f32 arrays and
    tensors map to F32, torch.bfloat16 tensors to BF16 in place (no copy)."""
    import ctypes as C
    import numpy as np
    import torch
    import paper_2505_15511_b200 as nb
    from paper_2505_15511_b200 import _native as N
    from paper_2505_15511_b200.api import _dataset
    assert [f[0] for f in N.DatasetView._fields_] == ["rows", "dims", "data", "location", "dtype"]
    assert C.sizeof(N.DatasetView) == 32
    v, _ = _dataset(np.zeros((3, 4), np.float64))
    assert (v.rows, v.dims, v.location, v.dtype) == (3, 4, N.HOST, N.F32)
    t = torch.zeros((5, 6), dtype=torch.bfloat16)
    v, keep = _dataset(t)
    assert (v.rows, v.dims, v.location, v.dtype) == (5, 6, N.HOST, N.BF16)
    assert v.data == t.data_ptr()
    hdr = open(os.path.join(ROOT, "include", "nomad_b200.h")).read()
    assert "#define NOMAD_B200_BF16 1" in hdr and "#define NOMAD_B200_F32 0" in hdr
