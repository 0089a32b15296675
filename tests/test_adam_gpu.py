"""GPU parity of the optimizer kernels (adam.hpp:67-313) through the C ABI: given identical
gradients, arena state after every pass is bit-identical to the reference — for the reference's
separate w/m/v arrays and for the row-interleaved layout (gss_arena.row_stride) the engine uses."""
import numpy as np
import pytest
import torch

import oracles as O
import paper_2509_15645_b200 as G

pytestmark = pytest.mark.gpu

GROUPS49 = [(0, 1, 5e-2), (1, 3, 2.5e-3), (4, 45, 1.25e-4)]
GROUPS10 = [(0, 3, 1.6e-4), (3, 3, 5e-3), (6, 4, 1e-3)]


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def make_pair(n, dim, groups, defer_max, rng, interleaved=False):
    ra = O.RefArena(n, dim, groups, defer_max)
    ga = G.Arena(n, dim, [G.GroupSpec(f"g{i}", c0, d, G.Hyperparams(lr)) for i, (c0, d, lr) in enumerate(groups)],
                 defer_max, interleaved=interleaved)
    w0 = rng.uniform(-1, 1, (n, dim)).astype(np.float32)
    ra.w[:] = w0
    ga.w.copy_(torch.from_numpy(w0))
    return ra, ga


def assert_same(ra, ga):
    assert np.array_equal(bits(ra.w), bits(ga.w.cpu().numpy()))
    assert np.array_equal(bits(ra.m), bits(ga.m.cpu().numpy()))
    assert np.array_equal(bits(ra.v), bits(ga.v.cpu().numpy()))
    assert np.array_equal(ra.counter, ga.counter.cpu().numpy())
    assert ra.step == ga.step


@pytest.mark.parametrize("interleaved", [False, True])
@pytest.mark.parametrize("defer_max", [0, 1, 7, 15, 40])
@pytest.mark.parametrize("n,dim,groups", [(3000, 49, GROUPS49), (2100, 10, GROUPS10), (777, 59, None)])
def test_deferred_schedule_bitwise(ref, defer_max, n, dim, groups, interleaved):
    rng = np.random.default_rng(defer_max * 1000 + n)
    if groups is None:
        groups = GROUPS10 + [(10 + c0, d, lr) for c0, d, lr in GROUPS49]
    ra, ga = make_pair(n, dim, groups, defer_max, rng, interleaved)
    for step in range(30):
        dens = 0.0 if step % 11 == 5 else rng.uniform(0.02, 0.3)
        ids = np.nonzero(rng.uniform(size=n) < dens)[0].astype(np.int32)
        rows = rng.normal(size=(ids.size, dim)).astype(np.float32)
        t_ref = ra.deferred(ids, rows, dim)
        t_gpu = G.deferred_update(ga, G.SparseGrads(torch.from_numpy(ids).cuda(), torch.from_numpy(rows).cuda(), dim))
        assert np.array_equal(t_ref, t_gpu.cpu().numpy())
        assert_same(ra, ga)


def test_strided_grads_with_col0_bitwise(ref):
    """The engine's geo update reads cols 0..9 of V x 59 rows; the non-geo one cols 10..58."""
    rng = np.random.default_rng(1)
    n = 1500
    ra, ga = make_pair(n, 49, GROUPS49, 15, rng)
    for _ in range(12):
        ids = np.nonzero(rng.uniform(size=n) < 0.2)[0].astype(np.int32)
        rows = rng.normal(size=(ids.size, 59)).astype(np.float32)
        ra.deferred(ids, rows, 59, 10)
        G.deferred_update(ga, G.SparseGrads(torch.from_numpy(ids).cuda(), torch.from_numpy(rows).cuda(), 59, 10))
        assert_same(ra, ga)


@pytest.mark.parametrize("interleaved", [False, True])
def test_dense_step_bitwise_and_fixed_point(ref, interleaved):
    rng = np.random.default_rng(2)
    n, dim = 999, 59
    groups = GROUPS10 + [(10 + c0, d, lr) for c0, d, lr in GROUPS49]
    ra, ga = make_pair(n, dim, groups, 0, rng, interleaved)
    for s in range(5):
        g = rng.normal(size=(n, dim)).astype(np.float32)
        ra.dense(g)
        G.adam_step_dense(ga, torch.from_numpy(g).cuda())
        assert_same(ra, ga)
    ra.dense(None)
    G.adam_step_dense(ga, None)
    assert_same(ra, ga)
    z = G.Arena(3, 4, [G.GroupSpec("all", 0, 4, G.Hyperparams(1e-3))], 0)
    G.adam_step_dense(z, None)  # zero state + zero grad is a fixed point (test_optim.cpp:29-36)
    assert torch.all(z.w == 0) and torch.all(z.m == 0) and torch.all(z.v == 0)


def test_max0_deferred_equals_dense_bitwise():
    """test_optim.cpp:110-133 on the device."""
    rng = np.random.default_rng(23)
    n, dim = 40, 7
    grp = [G.GroupSpec("all", 0, dim, G.Hyperparams(5e-3))]
    dense = G.Arena(n, dim, grp, 0)
    defer = G.Arena(n, dim, grp, 0)
    w0 = torch.from_numpy(rng.uniform(-2, 2, (n, dim)).astype(np.float32)).cuda()
    dense.w.copy_(w0)
    defer.w.copy_(w0)
    for _ in range(30):
        ids = np.nonzero(rng.uniform(size=n) < 0.3)[0].astype(np.int32)
        rows = rng.normal(size=(ids.size, dim)).astype(np.float32)
        g = np.zeros((n, dim), np.float32)
        g[ids] = rows
        G.adam_step_dense(dense, torch.from_numpy(g).cuda())
        t = G.deferred_update(defer, G.SparseGrads(torch.from_numpy(ids).cuda(), torch.from_numpy(rows).cuda(), dim))
        assert t.numel() == n
        assert torch.equal(dense.w, defer.w) and torch.equal(dense.m, defer.m) and torch.equal(dense.v, defer.v)


@pytest.mark.parametrize("interleaved", [False, True])
def test_restore_view_with_and_without_pending_bitwise(ref, interleaved):
    rng = np.random.default_rng(29)
    n, dim = 2000, 49
    ra, ga = make_pair(n, dim, GROUPS49, 6, rng, interleaved)
    for _ in range(9):
        ids = np.nonzero(rng.uniform(size=n) < 0.3)[0].astype(np.int32)
        rows = rng.normal(size=(ids.size, dim)).astype(np.float32)
        ra.deferred(ids, rows, dim)
        G.deferred_update(ga, G.SparseGrads(torch.from_numpy(ids).cuda(), torch.from_numpy(rows).cuda(), dim))
    pids = np.nonzero(rng.uniform(size=n) < 0.4)[0].astype(np.int32)
    prow = rng.normal(size=(pids.size, dim)).astype(np.float32)
    q = np.nonzero(rng.uniform(size=n) < 0.5)[0].astype(np.int32)
    pend = G.SparseGrads(torch.from_numpy(pids).cuda(), torch.from_numpy(prow).cuda(), dim)
    got = G.restore_view(ga, torch.from_numpy(q).cuda(), pend).cpu().numpy()
    assert np.array_equal(bits(got), bits(ra.restore(q, (pids, prow, dim, 0))))
    got0 = G.restore_view(ga, torch.from_numpy(q).cuda(), None).cpu().numpy()
    assert np.array_equal(bits(got0), bits(ra.restore(q)))
    assert_same(ra, ga)  # pure read
    # pending ids match the later deferred_update bitwise (test_optim.cpp:240-275)
    allids = torch.arange(n, dtype=torch.int32, device="cuda")
    fwd = G.restore_view(ga, allids, pend).cpu().numpy()
    touched = G.deferred_update(ga, pend).cpu().numpy()
    w = ga.w.cpu().numpy()
    assert np.array_equal(bits(w[touched]), bits(fwd[touched]))


@pytest.mark.parametrize("interleaved", [False, True])
def test_flush_equals_restore_and_reference(ref, interleaved):
    rng = np.random.default_rng(41)
    n, dim = 500, 49
    ra, ga = make_pair(n, dim, GROUPS49, 15, rng, interleaved)
    for _ in range(12):
        ids = np.nonzero(rng.uniform(size=n) < 0.3)[0].astype(np.int32)
        rows = rng.normal(size=(ids.size, dim)).astype(np.float32)
        ra.deferred(ids, rows, dim)
        G.deferred_update(ga, G.SparseGrads(torch.from_numpy(ids).cuda(), torch.from_numpy(rows).cuda(), dim))
    view = G.restore_view(ga, torch.arange(n, dtype=torch.int32, device="cuda"), None).clone()
    ra.flush()
    G.flush_deferred(ga)
    assert_same(ra, ga)
    assert torch.equal(ga.w, view)
    assert int(ga.counter.max()) == 0


def test_unsorted_ids_raise_invariant_violation():
    ga = G.Arena(100, 2, [G.GroupSpec("all", 0, 2, G.Hyperparams(1e-3))], 15)
    ids = torch.tensor([5, 3], dtype=torch.int32, device="cuda")
    rows = torch.ones((2, 2), device="cuda")
    with pytest.raises(G.InvariantViolation):
        G.deferred_update(ga, G.SparseGrads(ids, rows, 2))
    with pytest.raises(G.InvariantViolation):
        G.deferred_update(ga, G.SparseGrads(torch.tensor([1, 100], dtype=torch.int32, device="cuda"), rows, 2))


def test_bad_config_raises_config_error():
    with pytest.raises(G.ConfigError):
        G.Arena(10, 3, [G.GroupSpec("a", 0, 2, G.Hyperparams(1e-3))], 15)
    with pytest.raises(G.ConfigError):
        G.Arena(10, 2, [G.GroupSpec("a", 0, 2, G.Hyperparams(-1.0))], 15)
    with pytest.raises(G.ConfigError):
        G.Arena(10, 2, [G.GroupSpec("a", 0, 2, G.Hyperparams(1e-3))], 255)


def test_optim_bench_equivalence_on_device(ref):
    """acceptance criterion 1 on the device: 10% density, MAX=15 vs dense oracle <= 1e-4."""
    rng = O.Rng(42)
    n, dim, steps = 1000, 59, 500
    hp = [G.GroupSpec("all", 0, dim, G.Hyperparams(1e-3))]
    dense = G.Arena(n, dim, hp, 0)
    defer = G.Arena(n, dim, hp, 15)
    w0 = np.array([rng.uniform(-1.0, 1.0) for _ in range(n * dim)], np.float64).astype(np.float32).reshape(n, dim)
    dense.w.copy_(torch.from_numpy(w0))
    defer.w.copy_(torch.from_numpy(w0))
    nprng = np.random.default_rng(42)
    for _ in range(steps):
        ids = np.nonzero(nprng.uniform(size=n) < 0.10)[0].astype(np.int32)
        rows = nprng.normal(size=(ids.size, dim)).astype(np.float32)
        g = np.zeros((n, dim), np.float32)
        g[ids] = rows
        G.adam_step_dense(dense, torch.from_numpy(g).cuda())
        G.deferred_update(defer, G.SparseGrads(torch.from_numpy(ids).cuda(), torch.from_numpy(rows).cuda(), dim),
                          want_touched=False, check_invariants=False)
    G.flush_deferred(defer)
    dev = O.rel_err(dense.w.cpu().numpy(), defer.w.cpu().numpy()).max()
    assert dev <= 1e-4


@pytest.mark.parametrize("defer_max", [1, 15])
def test_engine_layout_interleaved_aligned_grads_bitwise(ref, defer_max):
    """The engine's layout: row-interleaved arena + 16-byte-aligned gradient rows (stride 52, the
    engine's gradient stage); padding columns of the gradient rows are never read as data."""
    rng = np.random.default_rng(77 + defer_max)
    n, dim = 5000, 49
    ra, ga = make_pair(n, dim, GROUPS49, defer_max, rng, interleaved=True)
    for step in range(40):
        dens = 0.0 if step % 13 == 7 else rng.uniform(0.02, 0.3)
        ids = np.nonzero(rng.uniform(size=n) < dens)[0].astype(np.int32)
        rows = rng.normal(size=(ids.size, 52)).astype(np.float32)
        rows[:, 49:] = np.nan  # padding: must never be read as data
        t_ref = ra.deferred(ids, rows, 52)
        t_gpu = G.deferred_update(ga, G.SparseGrads(torch.from_numpy(ids).cuda(), torch.from_numpy(rows).cuda(), 52))
        assert np.array_equal(t_ref, t_gpu.cpu().numpy())
        assert_same(ra, ga)
    ra.flush()
    G.flush_deferred(ga)
    assert_same(ra, ga)


@pytest.mark.parametrize("defer_max", [1, 15])
def test_host_tier_arena_passes_bitwise(ref, defer_max):
    """The pinned host tier (store.hpp:149-192): deferred passes, flush and the forwarding gather
    over host-resident rows (in place through the mapping; GSS_HOST_STAGING=1 stages them through
    HBM in chunks — a subprocess run below), bit-identical to the reference."""
    rng = np.random.default_rng(77 + defer_max)
    n, dim = 6000, 49
    ra = O.RefArena(n, dim, GROUPS49, defer_max)
    ga = G.Arena(n, dim, [G.GroupSpec(f"g{i}", c0, d, G.Hyperparams(lr)) for i, (c0, d, lr) in enumerate(GROUPS49)],
                 defer_max, interleaved=True, host=True)
    assert not ga.w.is_cuda and ga.counter.is_cuda
    w0 = rng.uniform(-1, 1, (n, dim)).astype(np.float32)
    ra.w[:] = w0
    ga.w.copy_(torch.from_numpy(w0))
    G.set_host_chunk_bytes(1024 * 156 * 4)  # 1024 rows per chunk
    try:
        for step in range(24):
            dens = 0.0 if step % 9 == 4 else rng.uniform(0.05, 0.6)
            ids = np.nonzero(rng.uniform(size=n) < dens)[0].astype(np.int32)
            rows = rng.normal(size=(ids.size, dim)).astype(np.float32)
            if step % 5 == 2:  # forwarding gather with this pass's gradients pending
                q = np.nonzero(rng.uniform(size=n) < 0.5)[0].astype(np.int32)
                pend = G.SparseGrads(torch.from_numpy(ids).cuda(), torch.from_numpy(rows).cuda(), dim)
                got = G.restore_view(ga, torch.from_numpy(q).cuda(), pend).cpu().numpy()
                assert np.array_equal(bits(got), bits(ra.restore(q, (ids, rows, dim, 0))))
            t_ref = ra.deferred(ids, rows, dim)
            t_gpu = G.deferred_update(ga, G.SparseGrads(torch.from_numpy(ids).cuda(), torch.from_numpy(rows).cuda(), dim))
            torch.cuda.synchronize()
            assert np.array_equal(t_ref, t_gpu.cpu().numpy())
            assert_same(ra, ga)
        q = np.arange(n, dtype=np.int32)
        got0 = G.restore_view(ga, torch.from_numpy(q).cuda(), None).cpu().numpy()
        assert np.array_equal(bits(got0), bits(ra.restore(q)))
        G.flush_deferred(ga)
        ra.flush()
        torch.cuda.synchronize()
        assert_same(ra, ga)
    finally:
        G.set_host_chunk_bytes(32 << 20)


def test_host_tier_staged_variant_bitwise():
    """The opt-in staged host-tier passes (GSS_HOST_STAGING=1: chunked gather -> device pass ->
    scatter on two streams) give the same bits as the reference (the test above in a subprocess)."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, GSS_HOST_STAGING="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                        f"{__file__}::test_host_tier_arena_passes_bitwise"], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))), timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("defer_max,n", [(1, 1), (6, 31), (15, 4099), (15, 40000)])
def test_engine_layout_gather_with_pending_bitwise(ref, defer_max, n):
    """The engine's forwarding gather layout: row-interleaved arena + 52-float pending gradient rows
    (restore_resolve_kernel + restore_walk_kernel): restored rows bitwise equal to the reference's
    restore_view with pending grads, at sizes around the 32-row batch boundary; padding columns of
    the gradient rows (NaN here) never read as data."""
    rng = np.random.default_rng(11 + defer_max + n)
    dim = 49
    ra, ga = make_pair(n, dim, GROUPS49, defer_max, rng, interleaved=True)
    for _ in range(defer_max + 3):
        ids = np.nonzero(rng.uniform(size=n) < 0.3)[0].astype(np.int32)
        rows = rng.normal(size=(ids.size, 52)).astype(np.float32)
        rows[:, 49:] = np.nan
        ra.deferred(ids, rows, 52)
        G.deferred_update(ga, G.SparseGrads(torch.from_numpy(ids).cuda(), torch.from_numpy(rows).cuda(), 52))
    assert_same(ra, ga)
    pids = np.nonzero(rng.uniform(size=n) < 0.4)[0].astype(np.int32)
    prow = rng.normal(size=(pids.size, 52)).astype(np.float32)
    prow[:, 49:] = np.nan
    q = np.nonzero(rng.uniform(size=n) < 0.6)[0].astype(np.int32)
    pend = G.SparseGrads(torch.from_numpy(pids).cuda(), torch.from_numpy(prow).cuda(), 52)
    got = G.restore_view(ga, torch.from_numpy(q).cuda(), pend).cpu().numpy()
    assert np.array_equal(bits(got), bits(ra.restore(q, (pids, prow, 52, 0))))
    got0 = G.restore_view(ga, torch.from_numpy(q).cuda(), None).cpu().numpy()
    assert np.array_equal(bits(got0), bits(ra.restore(q)))
    assert_same(ra, ga)
