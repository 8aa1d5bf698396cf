"""Multi-rank host logic on CPU (gloo, world_size 2): environment sharding and
the max-over-ranks throughput reduction used by bench.py."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2402_01181_b200.batch import shard, tile_shape


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_envs, out):
    import torch.distributed as dist
    from paper_2402_01181_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w, r, lr = D.world()
        assert (w, r, lr) == (world, rank, rank)
        mine = shard(n_envs, w, r)
        units = len(mine) * 1000.0          # particle-substeps done by this rank
        seconds = 1.0 + rank                # rank 1 is the slow one
        tp = D.throughput(units, seconds)
        gathered = [None] * world
        dist.all_gather_object(gathered, list(mine))
        out[rank] = (tp, gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_envs", [1024, 7])
def test_gloo_two_ranks_shard_and_throughput(n_envs):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n_envs, out), nprocs=world, join=True)
    tp0, envs = out[0]
    assert out[1][0] == tp0
    assert tp0 == pytest.approx(n_envs * 1000.0 / 2.0)  # total units / max time
    flat = [e for part in envs for e in part]
    assert flat == list(range(n_envs))                  # every env exactly once, contiguous


def test_shard_and_tiles_single_process():
    for n in (1, 5, 1024):
        for w in (1, 2, 3, 8):
            parts = [shard(n, w, r) for r in range(w)]
            assert sum(len(p) for p in parts) == n
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
    for n in (1, 3, 8, 100, 1024):
        t = tile_shape(n)
        assert t[0] * t[1] * t[2] >= n
        assert t[0] * t[1] * t[2] < 2 * n + 2


def _exchange_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2402_01181_b200.slab import TorchExchange, _neighbours
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = TorchExchange(None, rank, world, device="cpu")
        nbs = _neighbours(rank, world)
        # halo-record counts and payloads: rank r sends (r+1)*(nb+1) rows of value 100r+nb
        counts = ex.counts({nb: (rank + 1) * (nb + 1) for nb in nbs.values()})
        send = {nb: torch.full(((rank + 1) * (nb + 1), 3), 100.0 * rank + nb) for nb in nbs.values()}
        got = ex.payload(send, counts, 3, torch.float32)
        out[rank] = {nb: (counts[nb], float(got[nb][0, 0]) if counts[nb] else None, tuple(got[nb].shape))
                     for nb in nbs.values()}
    finally:
        dist.destroy_process_group()


def test_gloo_slab_neighbour_exchange_protocol():
    """The slab driver's point-to-point protocol (counts, then payloads) pairs
    every rank with its x-neighbours and delivers shapes/values intact."""
    world = 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_exchange_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        for nb, (cnt, val, shape) in out[r].items():
            assert cnt == (nb + 1) * (r + 1)
            assert val == 100.0 * nb + r
            assert shape == (cnt, 3)
    assert set(out[0]) == {1} and set(out[1]) == {0, 2} and set(out[2]) == {1}


def test_slab_partition():
    from paper_2402_01181_b200.slab import partition
    for res, ranks in ((1024, 8), (64, 3), (256, 2)):
        parts = partition(res, ranks)
        assert parts[0][0] == 0 and parts[-1][1] == res
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        assert all(lo % 4 == 0 and hi % 4 == 0 for lo, hi in parts)
        widths = [hi - lo for lo, hi in parts]
        assert max(widths) - min(widths) <= 4


def test_balanced_partition_narrow_scene():
    """a scene spanning x in [0.3, 0.7] cut for 4 and 8 ranks --
    every window holds particles, counts within a brick column of equal."""
    import numpy as np
    from paper_2402_01181_b200.slab import balanced_partition
    rng = np.random.default_rng(0)
    res = 1024
    base = np.floor(rng.uniform(0.3, 0.7, 2_000_000) * res - 0.5).astype(np.int64)
    for ranks in (2, 4, 8):
        parts = balanced_partition(base, res, ranks)
        assert parts[0][0] == 0 and parts[-1][1] == res
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        assert all(lo % 4 == 0 and hi % 4 == 0 and hi > lo for lo, hi in parts)
        counts = [int(((base >= lo) & (base < hi)).sum()) for lo, hi in parts]
        assert min(counts) > 0
        per_col = len(base) / (0.4 * res / 4)
        assert max(counts) - min(counts) <= 2 * per_col, counts
    # a scene occupying fewer columns than ranks cannot be cut
    import pytest
    from paper_2402_01181_b200.errors import ParameterError
    with pytest.raises(ParameterError):
        balanced_partition(np.full(100, 40), 64, 4)
