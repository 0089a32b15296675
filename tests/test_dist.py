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


# ---- image-parallel exchange plumbing, world_size 2 over gloo on CPU ----------

def _xchg_worker(rank, world, port, q):
    import torch

    from paper_2509_15645_b200 import imgpar as IP

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = IP.TorchExchange()
        # rank r sends (r + 1) * (j + 2) records to rank j; record bytes encode (src, dst, index)
        counts = [(rank + 1) * (j + 2) for j in range(world)]
        send = torch.zeros((sum(counts), 64), dtype=torch.uint8)
        off = 0
        for j, c in enumerate(counts):
            send[off: off + c, 0] = rank
            send[off: off + c, 1] = j
            send[off: off + c, 2] = torch.arange(c, dtype=torch.uint8)
            off += c
        recv, rcounts = ex.alltoallv(send, counts)
        # strip owner answers with 9 floats per received record: (src, index, own rank, ...)
        part = torch.zeros((recv.shape[0], 9), dtype=torch.float32)
        part[:, 0] = recv[:, 0].float()
        part[:, 1] = recv[:, 2].float()
        part[:, 2] = rank
        back, _ = ex.alltoallv(part, rcounts, recv_counts=counts)
        sums = ex.allgather_f64(torch.tensor([0.25 + rank], dtype=torch.float64))
        q.put((rank, counts, rcounts, recv.numpy(), back.numpy(), sums))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_imgpar_exchange():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xchg_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, counts, rcounts, recv, back, sums in res:
        assert rcounts == [(s + 1) * (rank + 2) for s in range(world)]
        # received rows: concatenated in source-rank order, each source's rows in its send order
        off = 0
        for s, c in enumerate(rcounts):
            assert (recv[off: off + c, 0] == s).all() and (recv[off: off + c, 1] == rank).all()
            assert np.array_equal(recv[off: off + c, 2], np.arange(c))
            off += c
        # answers come back in this rank's send order, strip by strip
        off = 0
        for j, c in enumerate(counts):
            assert (back[off: off + c, 0] == rank).all() and (back[off: off + c, 2] == j).all()
            assert np.array_equal(back[off: off + c, 1], np.arange(c))
            off += c
        assert sums == [0.25, 1.25]


def test_strip_bounds_and_loss_arithmetic():
    from paper_2509_15645_b200 import imgpar as IP

    for pw in (0, 1, 15, 16, 17, 48, 1920, 3840):
        for n in (1, 2, 3, 8):
            b = IP.strip_bounds(7, pw, n)
            assert len(b) == n + 1 and b[0] == 7 and b[-1] == 7 + pw
            assert all(x <= y for x, y in zip(b, b[1:]))
            assert all((y - 7) % 16 == 0 or y == 7 + pw for y in b[1:-1])  # cuts on tile boundaries
            w = [y - x for x, y in zip(b, b[1:])]
            assert max(w) - min(w) <= 16 or pw < 16 * n
    # (float)(sum) * (1/(float)norm) in IEEE single, as the device loss_final kernel
    s = [1234.5678901234, 0.0009876, 77.125]
    want = np.float32(sum(s)) * (np.float32(1.0) / np.float32(6220800.0))
    assert IP.loss_from_sums(s, 6220800) == float(want)
    # the same arithmetic on tensors (device path, no host round trip): identical float32
    import torch
    for parts in (s, [3.0], [1e-3, 2e-3, 5.5, 1e9, 7.0, 0.25, 0.5, 0.125]):
        got = IP.loss_from_sums_dev(torch.tensor(parts, dtype=torch.float64), 6220800)
        assert got.dtype == torch.float32 and float(got) == IP.loss_from_sums(parts, 6220800)
