"""CPU, world_size 2 (gloo): the multi-rank host path of the epoch loop.

Each rank owns workers [r W/2, (r+1) W/2) of the shard plan the engine uses
(nomad_b200_plan), computes its clusters' means over its own points only,
packs them into the engine's slot layout and all-gathers; every rank must
then hold exactly gather_means() of the full layout (optimizer.hpp:149-176,
:411-442: one message per worker, no positions cross ranks)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, W, out_q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_2505_15511_b200 as nb
    from oracle import Oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("port")
    rng = np.random.default_rng(3)
    n, C = 4000, 12
    a = rng.integers(0, C, n).astype(np.uint32)
    layout = rng.normal(size=(n, 2)) * 5
    c2w, slots = nb.shard_plan(a, C, W, world)
    nwl = W // world
    mine = (c2w[a] >= rank * nwl) & (c2w[a] < (rank + 1) * nwl)
    # owned clusters' means from this rank's points only, ascending point id
    send = np.zeros((slots.shape[1], 2))
    for q, c in enumerate(slots[rank]):
        if c == 0xFFFFFFFF:
            continue
        idx = np.nonzero(mine & (a == c))[0]
        assert len(idx) == np.count_nonzero(a == c)  # the cluster lives on one rank
        acc = np.zeros(2)
        for i in idx:  # sequential, as gather_means accumulates
            acc[0] += layout[i, 0]
            acc[1] += layout[i, 1]
        send[q] = acc / len(idx)
    recv = [torch.zeros(slots.shape[1], 2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(recv, torch.from_numpy(send))
    means = np.full((C, 2), np.nan)
    for r in range(world):
        for q, c in enumerate(slots[r]):
            if c != 0xFFFFFFFF:
                means[c] = recv[r][q].numpy()
    ref = orc.gather_means(layout, a, C)
    out_q.put((rank, bool(np.array_equal(means, ref)), int(np.count_nonzero(c2w >= 0))))
    dist.destroy_process_group()


@pytest.mark.parametrize("W", [2, 4])
def test_two_rank_means_allgather_is_exact(W):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, W, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _, _ in res) == [0, 1]
    assert all(ok for _, ok, _ in res), res


def test_plan_matches_reference_shard_clusters(port):
    """The engine's LPT plan equals shard_clusters of the reference port."""
    import paper_2505_15511_b200 as nb
    rng = np.random.default_rng(0)
    for C, W in [(8, 4), (13, 3), (64, 8), (5, 5)]:
        a = rng.integers(0, C, 5000).astype(np.uint32)
        c2w, slots = nb.shard_plan(a, C, W, 1)
        rc2w, _ = port.shard_clusters(a, C, W)
        assert np.array_equal(c2w, rc2w)
        got = sorted(int(c) for c in slots.ravel() if c != 0xFFFFFFFF)
        assert got == list(range(C))
    with pytest.raises(nb.NomadError) as e:
        nb.shard_plan(np.zeros(10, np.uint32), 2, 3, 1)
    assert e.value.kind == "Parameter"
