"""N>1 host logic on CPU with world_size-2 gloo: id-range shards tile [0, n)
exactly, max-over-ranks timing, and the sharded cull — each rank culls its contiguous id shard,
ids are concatenated in shard order — equals the unsharded cull bit for bit (the oracle C
restatement computes the per-shard culls here: there is no GPU on this host)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracles as O
from paper_2509_15645_b200 import dist as D


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # timing aggregation
        ms = D.max_over_ranks(10.0 + rank)
        # sharded cull
        rng = np.random.default_rng(5)
        n = 40_000
        rows = np.zeros((n, 10), np.float32)
        rows[:, 0:3] = rng.uniform(-3, 3, (n, 3))
        rows[:, 3:6] = rng.uniform(-7, 1, (n, 3))
        qq = rng.normal(size=(n, 4))
        rows[:, 6:10] = qq / np.linalg.norm(qq, axis=1, keepdims=True)
        cam = O.look_at([0.3, 0.2, -4.0], [0, 0, 0], 300.0, 300.0, 320, 240, 0.5, 8.0)
        lo, hi = D.id_range(n, rank, world)
        local = O.orc_cull(np.ascontiguousarray(rows[lo:hi]), cam, [0, 320, 0, 240])
        glob = D.gather_ids(local, lo)
        q.put((rank, ms, (lo, hi), glob))
    finally:
        dist.destroy_process_group()


def test_id_range_tiles_exactly():
    for n in (0, 1, 7, 100, 1_000_003):
        for w in (1, 2, 3, 8):
            spans = [D.id_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_gloo_world2_sharded_cull_and_timing(orc):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] == 11.0 for r in res)  # max over ranks
    glob = res[0][3]
    assert np.array_equal(glob, res[1][3])
    # unsharded reference cull of the same rows
    rng = np.random.default_rng(5)
    n = 40_000
    rows = np.zeros((n, 10), np.float32)
    rows[:, 0:3] = rng.uniform(-3, 3, (n, 3))
    rows[:, 3:6] = rng.uniform(-7, 1, (n, 3))
    qq = rng.normal(size=(n, 4))
    rows[:, 6:10] = qq / np.linalg.norm(qq, axis=1, keepdims=True)
    cam = O.look_at([0.3, 0.2, -4.0], [0, 0, 0], 300.0, 300.0, 320, 240, 0.5, 8.0)
    assert np.array_equal(glob, O.orc_cull(rows, cam, [0, 320, 0, 240]))
    assert D.aggregate_throughput([3, 3], 500.0) == 12.0
