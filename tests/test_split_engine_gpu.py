"""Split-camera execution in the B200 OffloadEngine against the reference engine given the same
SplitTable (engine.hpp:62-68, 266-273, 355-371; splitter.hpp:85-123).

A split camera is culled as two closed viewports [0, s] and [s, W] whose sorted union is the
plan's id list; it is rendered as two sub-passes (each loss normalised by the full image, loss =
left + right) and the two gradient buffers are aggregated over the union, left added first. The
device path must give the reference's valid counts exactly, the first loss bit for bit (each
sub-pass forward + L1 is bit-exact), and the trajectory within the per-step tolerance.
"""
import numpy as np
import pytest
import torch

import oracles as O
import paper_2509_15645_b200 as G
from paper_2509_15645_b200 import evalsplit as ES

pytestmark = pytest.mark.gpu


def scene(n=220, cams=6, w=36, h=28, seed=91):
    cfg = G.SynthConfig(n=n, cams=cams, width=w, height=h, seed=seed)
    truth, cams_r, gts = O.ref_synth(cfg, with_gt=True)
    start = truth.copy()
    start[:, 10] = np.float32(np.log(0.1) - np.log(0.9))
    start[:, 14:] = 0.0
    return start, cams_r, gts


def engine(start, cams_r, gts, **kw):
    cams = [G.camera_from_bytes(c.tobytes()) for c in cams_r]
    return G.OffloadEngine(start, cams, gts, **kw)


SPLITS = [(1, 18), (0, 0), (1, 1), (1, 35), (0, 0), (1, 11)]


@pytest.mark.parametrize("defer,pipelined", [(15, True), (0, False), (15, False)])
def test_split_engine_tracks_reference(ref, defer, pipelined):
    start, cams, gts = scene()
    ours = engine(start, cams, gts, optim=G.OptimConfig(defer_max=defer), pipelined=pipelined, splits=SPLITS)
    theirs = O.RefEngine(start, cams, gts, defer_max=defer, pipelined=pipelined, splits=SPLITS)
    l1, v1 = ours.run(18)
    l2, v2 = theirs.run(18)
    assert np.array_equal(v1, v2)
    assert l1[0] == l2[0]  # two bit-exact sub-pass losses summed in float
    dev = float(O.rel_err(l1, l2).max())
    snap = float(O.rel_err(ours.snapshot(), theirs.snapshot()).max())
    print(f"split engine: loss dev {dev:.3e}, snapshot dev {snap:.3e}")
    assert dev <= 1e-4 and snap <= 1e-4
    s1, s2 = ours.state(), theirs.state()
    assert np.array_equal(s1["ng_counter"], s2["ng_counter"])
    n1, c1 = ours.accum()
    n2, c2 = theirs.accum()
    assert np.array_equal(c1, c2)
    assert float(O.rel_err_floor(n1, n2, 1e-3 * max(n2.max(), 1e-30)).max()) <= 1e-2


def test_split_serial_equals_pipelined_bitwise():
    start, cams, gts = scene(seed=17)
    a = engine(start, cams, gts, pipelined=False, splits=SPLITS)
    b = engine(start, cams, gts, pipelined=True, splits=SPLITS)
    la, va = a.run(20)
    lb, vb = b.run(20)
    assert np.array_equal(la.view(np.uint32), lb.view(np.uint32))
    assert np.array_equal(va, vb)
    assert np.array_equal(a.snapshot().view(np.uint32), b.snapshot().view(np.uint32))


def test_split_union_equals_whole_cull():
    """The union of the two closed-viewport culls is the whole-view cull: same valid counts as the
    unsplit engine on the first iteration of every camera."""
    start, cams, gts = scene(seed=5)
    a = engine(start, cams, gts, splits=[(1, 1 + 5 * i) for i in range(len(cams))])
    b = engine(start, cams, gts)
    _, va = a.run(len(cams))
    _, vb = b.run(len(cams))
    assert va[0] == vb[0]


def test_split_table_from_search_matches_reference_engine(ref):
    """compute_split_points (device culls) -> SplitTable -> engine, against the reference's own
    compute_split_points + OffloadEngine (the trainer's offload path, trainer.hpp)."""
    start, cams_r, gts = scene(n=400, w=40, h=30, seed=123)
    cams = [G.camera_from_bytes(c.tobytes()) for c in cams_r]
    geo = torch.from_numpy(np.ascontiguousarray(start[:, :10])).cuda()
    table = ES.compute_split_points(geo, start.shape[0], cams, 0.05)
    assert any(e.split for e in table)
    ref_table, _ = O.ref_compute_split_points(np.ascontiguousarray(start[:, :10]), cams_r, 0.05)
    pairs = [(int(e.split), int(e.column)) for e in table]
    assert pairs == [(int(r[0]), int(r[1])) for r in ref_table]
    ours = G.OffloadEngine(start, cams, gts, splits=table)
    theirs = O.RefEngine(start, cams_r, gts, pipelined=True, splits=pairs)
    l1, v1 = ours.run(12)
    l2, v2 = theirs.run(12)
    assert np.array_equal(v1, v2)
    assert float(O.rel_err(l1, l2).max()) <= 1e-4


def test_split_table_validation():
    start, cams, gts = scene(n=50, cams=2, seed=3)
    e = engine(start, cams, gts)
    with pytest.raises(G.ConfigError):
        e.set_splits([(1, 0), (0, 0)])  # column must lie in (0, W)
    with pytest.raises(G.ConfigError):
        e.set_splits([(1, 36), (0, 0)])
    with pytest.raises(G.ConfigError):
        e.set_splits([(1, 5)])  # one entry per camera
    e.set_splits([(1, 5), (0, 0)])
    losses, _ = e.run(2)
    assert np.all(np.isfinite(losses))
