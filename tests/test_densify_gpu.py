"""Densification on the device against the reference's plan_densify /
apply_densify (trainer.hpp:166-213, engine.hpp:116-163):

  * given the same snapshot and statistics, the plan is bit-identical: survivors (ascending ids),
    clone / split / prune counts and every child row (split children draw the reference Rng
    stream with glibc libm: the host computes them), including opacities and scales placed on the
    float neighbours of the prune / clone thresholds;
  * the engine's event keeps survivors' stored parameters, optimizer state and counters, appends the
    children with zero state, resets the statistics, and trains on; against the reference engine
    running the same schedule the population and the trained parameters agree within the step
    tolerance.
"""
import numpy as np
import pytest
import torch

import oracles as O
import paper_2509_15645_b200 as G

pytestmark = pytest.mark.gpu

DCFG = G.DensifyConfig()
DARR = [DCFG.grad_threshold, DCFG.percent_dense, DCFG.opacity_prune, DCFG.split_scale_divisor]


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def random_population(seed, n, extent):
    rng = np.random.default_rng(seed)
    rows = np.zeros((n, 59), np.float32)
    rows[:, 0:3] = rng.uniform(-1, 1, (n, 3))
    lim = np.log(DCFG.percent_dense * extent)
    rows[:, 3:6] = rng.uniform(lim - 1.5, lim + 1.5, (n, 3))
    q = rng.normal(size=(n, 4))
    rows[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    rows[:, 10] = rng.uniform(-8, 3, n)
    rows[:, 11:] = rng.normal(0, 0.3, (n, 48))
    # exact threshold neighbourhoods: opacity logits and max log-scales a few ulps around the cuts
    t = np.float32(np.log(DCFG.opacity_prune / (1 - DCFG.opacity_prune)))
    k = min(64, n // 8)
    near = t + np.arange(-k // 2, k // 2).astype(np.float32) * np.spacing(t)
    rows[:k, 10] = near
    s = np.float32(lim)
    rows[k:2 * k, 3] = s + np.arange(-k // 2, k // 2).astype(np.float32) * np.spacing(s)
    rows[k:2 * k, 4:6] = s - 1
    cnt = rng.integers(0, 6, n).astype(np.int32)
    norm = rng.uniform(0, 2 * DCFG.grad_threshold, n) * cnt
    norm[2 * k:3 * k] = DCFG.grad_threshold * cnt[2 * k:3 * k]  # avg exactly at the threshold
    rows[2 * k:3 * k, 10] = 2.0
    rows[k:2 * k, 10] = 2.0
    norm[k:2 * k] = 3 * DCFG.grad_threshold * np.maximum(cnt[k:2 * k], 1)
    cnt[k:2 * k] = np.maximum(cnt[k:2 * k], 1)
    return rows, norm, cnt


@pytest.mark.parametrize("seed,n,extent", [(1, 3000, 1.0), (2, 20000, 2.5), (3, 257, 0.3)])
def test_plan_equals_reference(ref, seed, n, extent):
    rows, norm, cnt = random_population(seed, n, extent)
    ev_seed = 0x1234 ^ (0x9E37 * seed)
    rs, rk, rc = O.ref_plan_densify(rows, norm, cnt, DARR, extent, ev_seed)
    gs, gk, gc = G.plan_densify(torch.from_numpy(rows).cuda(), torch.from_numpy(norm).cuda(),
                                torch.from_numpy(cnt).cuda(), DCFG, extent, ev_seed)
    assert [gc[k] for k in ("survivors", "children", "clones", "splits", "pruned")] == rc.tolist()
    assert rc[2] > 0 and rc[3] > 0 and rc[4] > 0  # every branch exercised
    assert np.array_equal(gs.cpu().numpy(), rs)
    assert np.array_equal(bits(gk.cpu().numpy()), bits(rk))


def test_engine_densify_semantics_and_reference():
    cfg = G.SynthConfig(n=3000, cams=6, width=64, height=48, seed=5)
    truth, cams = G.synth_scene_params(cfg)
    gts = np.stack([G.render_view(torch.from_numpy(truth).cuda(), c, 3).cpu().numpy() for c in cams])
    start = truth.copy()
    start[:, 10] = np.float32(np.log(0.1 / 0.9))
    start[:, 14:] = 0.0
    dcfg = G.DensifyConfig(grad_threshold=2e-5)  # small threshold: clones and splits happen
    e = G.OffloadEngine(start, cams, gts, pipelined=True)
    e.run(6)
    before = e.state()
    snap = e.snapshot()
    norm, cnt = e.accum()
    rs, rk, rc = O.ref_plan_densify(snap, norm, cnt, [dcfg.grad_threshold, dcfg.percent_dense, dcfg.opacity_prune,
                                                      dcfg.split_scale_divisor], 1.0, 99)
    counts = e.densify(dcfg, 1.0, 99)
    assert [counts[k] for k in ("survivors", "children", "clones", "splits", "pruned")] == rc.tolist()
    assert counts["children"] > 0
    after = e.state()
    ns = len(rs)
    assert np.array_equal(bits(after["geo_w"][:ns]), bits(before["geo_w"][rs]))
    for k in ("ng_w", "ng_m", "ng_v"):
        assert np.array_equal(bits(after[k][:ns]), bits(before[k][rs])), k
    assert np.array_equal(after["ng_counter"][:ns], before["ng_counter"][rs])
    assert np.array_equal(bits(after["geo_w"][ns:]), bits(rk[:, :10]))
    assert np.array_equal(bits(after["ng_w"][ns:]), bits(rk[:, 10:]))
    assert not after["ng_m"][ns:].any() and not after["ng_v"][ns:].any() and not after["ng_counter"][ns:].any()
    n2, c2 = e.accum()
    assert not n2.any() and not c2.any()
    losses, _ = e.run(3)
    assert np.all(np.isfinite(losses))
    # the reference engine through the same schedule
    r = O.RefEngine(start, np.stack([O.cam_from_struct(c) for c in cams]), gts, pipelined=True)
    r.run(6)
    rc2 = r.densify([dcfg.grad_threshold, dcfg.percent_dense, dcfg.opacity_prune, dcfg.split_scale_divisor],
                    1.0, 99)
    assert rc2.tolist() == rc.tolist()  # statistics within tolerance: same decisions here
    rl, _ = r.run(3)
    assert np.allclose(losses, rl, rtol=1e-4, atol=1e-6)
    dev = O.rel_err(e.snapshot(), r.snapshot()).max()
    assert dev <= 1e-3, dev
    e.close()
