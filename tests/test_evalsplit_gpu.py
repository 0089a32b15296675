"""Evaluation and split search on the device against the reference:
compute_split_points (splitter.hpp:31-81) gives the identical table (every evaluation is an exact
device cull); psnr_over_views (trainer.hpp:131-145) agrees to fp64 summation order (images are
bit-identical); balanced strips for image-parallel rendering keep the split render bit-exact."""
import math

import numpy as np
import pytest
import torch

import oracles as O
import paper_2509_15645_b200 as G
from paper_2509_15645_b200 import evalsplit as ES
from paper_2509_15645_b200 import imgpar as IP

pytestmark = pytest.mark.gpu


def scene(seed, n, w, h, cams=6):
    cfg = G.SynthConfig(seed=seed, n=n, cams=cams, width=w, height=h)
    return G.synth_scene_params(cfg)


@pytest.mark.parametrize("mem_limit", [0.0, 0.2, 0.5])
def test_split_points_equal_reference(ref, mem_limit):
    rows, cams = scene(11, 6000, 96, 64, cams=8)
    geo = np.ascontiguousarray(rows[:, :10])
    want, ratio = O.ref_compute_split_points(geo, np.stack([O.cam_from_struct(c) for c in cams]), mem_limit)
    got = ES.compute_split_points(torch.from_numpy(geo).cuda(), geo.shape[0], cams, mem_limit)
    for i, e in enumerate(got):
        assert [int(e.split), e.column, e.left_count, e.right_count, e.search_evals] == want[i].tolist(), i
        assert e.used_ratio == ratio[i]


def test_psnr_over_views_matches_reference(ref):
    rows, cams = scene(3, 2000, 64, 48)
    truth = torch.from_numpy(rows).cuda()
    gts = [G.render_view(truth, c, 3) for c in cams]
    start = rows.copy()
    start[:, 10] -= 0.5
    start[:, 14:] *= 0.5
    db, exact = ES.psnr_over_views(torch.from_numpy(start).cuda(), cams, gts)
    rdb, rexact = O.ref_psnr_over_views(start, np.stack([O.cam_from_struct(c) for c in cams]),
                                        np.stack([g.cpu().numpy() for g in gts]))
    assert not exact and not rexact
    assert abs(db - rdb) <= 1e-9 * abs(rdb), (db, rdb)
    db2, exact2 = ES.psnr_over_views(truth, cams, gts)
    assert exact2 and math.isinf(db2)


def test_balanced_strips_render_bit_exact():
    rows, cams = scene(17, 20000, 200, 120)
    t = torch.from_numpy(rows).cuda()
    geo, ng = t[:, :10].contiguous(), t[:, 10:].contiguous()
    cam = cams[0]
    vp = G.viewport_full(200, 120)

    def upto(c):
        return int(G.frustum_cull(geo, geo.shape[0], cam, G.GssViewport(0.0, float(c), 0.0, 120.0)).numel())

    b = ES.balanced_strip_bounds(upto, 0, 200, 4)
    assert b[0] == 0 and b[-1] == 200 and all(x <= y for x, y in zip(b, b[1:]))
    assert all(x % 16 == 0 for x in b[1:-1])
    ids = G.frustum_cull(geo, geo.shape[0], cam, vp)
    sc = G.RenderScene(ids=ids, geo=geo, nongeo=ng)
    fw = G.rasterize_forward(sc, cam, vp)
    st, send, counts = IP.owner_project(sc, cam, vp, b)
    parts, off = [], 0
    for k in range(4):
        recv = send[off: off + counts[k]]
        off += counts[k]
        parts.append(IP.strip_forward(recv, cam, IP.strip_viewport(vp, b, k), (0.0, 0.0, 0.0), None, 0).image)
    img = torch.cat(parts, dim=1)
    assert torch.equal(img, fw.image)


@pytest.mark.parametrize("m,knn,colors", [(1, 3, False), (2, 3, True), (5000, 3, True), (3001, 8, False)])
def test_init_gaussians_equals_reference(ref, m, knn, colors):
    """init_gaussians (scene.hpp:146-195): exact O(M^2) kNN on the device."""
    rng = np.random.default_rng(m + knn)
    pos = rng.uniform(-1, 1, (m, 3)).astype(np.float32)
    if m > 10:
        pos[5] = pos[3]  # duplicate points: zero distances and ties
        pos[7] = pos[3]
    col = rng.uniform(0, 1, (m, 3)).astype(np.float32) if colors else None
    want = O.ref_init_gaussians(pos, col, knn)
    got = G.init_gaussians(pos, col, knn)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
