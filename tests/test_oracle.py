"""Pins the CPU oracle (oracle/gss_oracle.c) against the reference itself (oracle/_ref, the
unmodified reference headers) and against the committed golden fixtures (tests/golden/).
CPU only; these are the checks that make the oracle trustworthy as the GPU parity checker."""
import math
from pathlib import Path

import numpy as np
import pytest

import oracles as O

GOLDEN = Path(__file__).resolve().parent / "golden"


def _bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


# ---- expf: the one parity-relevant libm call (render.hpp:105, 348, 374) ----------------------

def test_expf_restatement_matches_host_libm_on_a_dense_sample(orc, ref):
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(-110, 95, 200000), np.array([float.fromhex("0x1.04845ep+5"), -float.fromhex("0x1.f8cbb2p+5"), 0.0, -0.0, 88.72,
                                                                  88.73, -103.97, -103.98, np.inf, -np.inf])])
    xs = xs.astype(np.float32)
    a = np.array([orc.orc_expf(float(x)) for x in xs], np.float32)
    b = np.array([ref.ref_expf(float(x)) for x in xs], np.float32)
    assert np.array_equal(_bits(a), _bits(b))


def test_expf_golden_vectors(orc):
    g = np.load(GOLDEN / "expf.npz")
    a = np.array([orc.orc_expf(float(x)) for x in g["x"]], np.float32)
    assert np.array_equal(_bits(a), _bits(g["y"]))


# ---- projection + cull (render.hpp:90-148, 243-260) ------------------------------------------

def test_project_matches_reference(orc, ref):
    rng = O.Rng(13)
    for trial in range(20):
        cam = O.look_at([rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(-4, -2)], [0, 0, 0], 80.0, 80.0, 64, 64,
                        0.1, 100.0)
        rows, _ = O.acceptance5_scene(rng, 50)
        for r in rows:
            a = np.zeros(8, np.float32)
            b = np.zeros(8, np.float32)
            orc.orc_project_geo(r.ctypes.data, cam.ctypes.data, 0.3, a.ctypes.data)
            ref.ref_project_geo(r.ctypes.data, cam.ctypes.data, 0.3, b.ctypes.data)
            assert np.array_equal(_bits(a), _bits(b))


def test_cull_depth_plane_exclusions(orc):
    """test_render.cpp:183-196."""
    cam = O.basic_cam(64, 64, 60.0, 0.5, 10.0)
    rows = np.array([[0, 0, z, -2, -2, -2, 1, 0, 0, 0] for z in (11.0, 0.4, 5.0, -3.0)], np.float32)
    assert list(O.orc_cull(rows, cam, [0, 64, 0, 64])) == [2]


def test_cull_center_always_kept(orc):
    """test_render.cpp:198-203."""
    cam = O.basic_cam(32, 32, 40.0)
    rows = np.array([[0, 0, 3, -4, -4, -4, 1, 0, 0, 0]], np.float32)
    assert list(O.orc_cull(rows, cam, [0, 32, 0, 32])) == [0]


def test_cull_acceptance5_scenes_equal_reference(orc, ref):
    """acceptance.cpp:215-257: 50 scene/camera pairs, exact set equality."""
    rng = O.Rng(77)
    for _ in range(50):
        rows, cam = O.acceptance5_scene(rng)
        vp = [0, 48, 0, 40]
        assert np.array_equal(O.orc_cull(rows, cam, vp), O.ref_cull(rows, cam, vp))


def test_cull_golden(orc):
    g = np.load(GOLDEN / "cull.npz")
    for k in range(int(g["n_cases"])):
        got = O.orc_cull(g[f"rows{k}"], g[f"cam{k}"], g[f"vp{k}"])
        assert np.array_equal(got, g[f"ids{k}"]), k


def test_cull_large_random_scene_equals_reference(orc, ref):
    rng = np.random.default_rng(5)
    n = 200_000
    rows = np.zeros((n, 10), np.float32)
    rows[:, 0:3] = rng.uniform(-3, 3, (n, 3))
    rows[:, 3:6] = rng.uniform(-6, 0.5, (n, 3))
    q = rng.normal(size=(n, 4))
    rows[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    cam = O.look_at([0.3, 0.2, -4.0], [0, 0, 0], 300.0, 300.0, 320, 240, 0.5, 8.0)
    for vp in ([0, 320, 0, 240], [0, 160, 0, 240], [160, 320, 0, 240]):
        assert np.array_equal(O.orc_cull(rows, cam, vp), O.ref_cull(rows, cam, vp))


# ---- optimizer (adam.hpp:67-313) -------------------------------------------------------------

def test_luts_match_reference(orc, ref):
    for t in (1, 2, 3, 16, 100, 30000):
        for md in (0, 3, 15, 40):
            a, sa = O.ref_luts(1e-3, t, md)
            b = [np.zeros(md + 1, np.float32) for _ in range(5)]
            sb = np.zeros(5, np.float32)
            orc.orc_build_luts(1e-3, 0.9, 0.999, 1e-8, t, md, *[x.ctypes.data for x in b], sb.ctypes.data)
            for x, y in zip(a, b):
                assert np.array_equal(_bits(x), _bits(y))
            assert np.array_equal(_bits(sa), _bits(sb))


class OrcArena:
    def __init__(self, n, dim, groups, defer_max):
        import ctypes as C

        class S(C.Structure):
            _fields_ = [("n", C.c_int64), ("dim", C.c_int), ("ngroups", C.c_int), ("col0", C.c_int * 8),
                        ("gdim", C.c_int * 8), ("lr", C.c_double * 8), ("b1", C.c_double), ("b2", C.c_double),
                        ("eps", C.c_double), ("defer_max", C.c_int), ("step", C.c_int64), ("w", C.c_void_p),
                        ("m", C.c_void_p), ("v", C.c_void_p), ("counter", C.c_void_p)]

        self.w = np.zeros((n, dim), np.float32)
        self.m = np.zeros((n, dim), np.float32)
        self.v = np.zeros((n, dim), np.float32)
        self.counter = np.zeros(max(n, 1), np.uint8)
        s = S()
        s.n, s.dim, s.ngroups = n, dim, len(groups)
        for i, (c0, d, lr) in enumerate(groups):
            s.col0[i], s.gdim[i], s.lr[i] = c0, d, lr
        s.b1, s.b2, s.eps, s.defer_max, s.step = 0.9, 0.999, 1e-8, defer_max, 0
        s.w, s.m, s.v, s.counter = self.w.ctypes.data, self.m.ctypes.data, self.v.ctypes.data, self.counter.ctypes.data
        self.s = s
        self.C = C

    def deferred(self, ids, rows, stride):
        ids = np.ascontiguousarray(ids, np.int32)
        rows = np.ascontiguousarray(rows, np.float32) if rows is not None else np.zeros(1, np.float32)
        t = np.zeros(max(self.w.shape[0], 1), np.int32)
        k = O.orc().orc_deferred_update(self.C.byref(self.s), ids.size, ids.ctypes.data, rows.ctypes.data, stride, 0,
                                        t.ctypes.data)
        return t[:k].copy()

    def dense(self, grads):
        O.orc().orc_adam_step_dense(self.C.byref(self.s), None if grads is None else grads.ctypes.data)

    def restore(self, ids, pending):
        ids = np.ascontiguousarray(ids, np.int32)
        out = np.zeros((max(ids.size, 1), self.w.shape[1]), np.float32)
        if pending is None:
            O.orc().orc_restore_view(self.C.byref(self.s), ids.size, ids.ctypes.data, 0, 0, None, None, 0, 0,
                                     out.ctypes.data)
        else:
            pids, prows = np.ascontiguousarray(pending[0], np.int32), np.ascontiguousarray(pending[1], np.float32)
            O.orc().orc_restore_view(self.C.byref(self.s), ids.size, ids.ctypes.data, 1, pids.size, pids.ctypes.data,
                                     prows.ctypes.data, self.w.shape[1], 0, out.ctypes.data)
        return out[: ids.size]

    def flush(self):
        O.orc().orc_flush_deferred(self.C.byref(self.s))


def test_adam_schedule_bitwise_vs_reference(orc, ref):
    """Random sparse schedule (bench.hpp:41-114 style) through deferred_update, restore_view with
    pending, flush_deferred and adam_step_dense: bit-identical state at every step."""
    rng = np.random.default_rng(17)
    n, dim = 300, 49
    groups = [(0, 1, 5e-2), (1, 3, 2.5e-3), (4, 45, 1.25e-4)]
    for defer in (0, 3, 15):
        ra = O.RefArena(n, dim, groups, defer)
        oa = OrcArena(n, dim, groups, defer)
        w0 = rng.uniform(-1, 1, (n, dim)).astype(np.float32)
        ra.w[:] = w0
        oa.w[:] = w0
        for step in range(40):
            ids = np.nonzero(rng.uniform(size=n) < 0.1)[0].astype(np.int32)
            rows = rng.normal(size=(ids.size, dim)).astype(np.float32)
            if step % 7 == 3:
                pids = np.nonzero(rng.uniform(size=n) < 0.2)[0].astype(np.int32)
                prow = rng.normal(size=(pids.size, dim)).astype(np.float32)
                q = np.nonzero(rng.uniform(size=n) < 0.3)[0].astype(np.int32)
                assert np.array_equal(_bits(ra.restore(q, (pids, prow, dim, 0))), _bits(oa.restore(q, (pids, prow))))
                assert np.array_equal(_bits(ra.restore(q)), _bits(oa.restore(q, None)))
            ta = ra.deferred(ids, rows, dim)
            tb = oa.deferred(ids, rows, dim)
            oa.s.step = ra.step
            assert np.array_equal(ta, tb)
            for x, y in ((ra.w, oa.w), (ra.m, oa.m), (ra.v, oa.v)):
                assert np.array_equal(_bits(x), _bits(y))
            assert np.array_equal(ra.counter, oa.counter[:n])
        ra.flush()
        oa.flush()
        assert np.array_equal(_bits(ra.w), _bits(oa.w))
        g = rng.normal(size=(n, dim)).astype(np.float32)
        ra.dense(g)
        oa.dense(g)
        assert np.array_equal(_bits(ra.w), _bits(oa.w))


def test_deferred_unsorted_ids_is_invariant_violation(orc):
    oa = OrcArena(10, 2, [(0, 2, 1e-3)], 15)
    ids = np.array([5, 3], np.int32)
    rows = np.ones((2, 2), np.float32)
    k = O.orc().orc_deferred_update(oa.C.byref(oa.s), 2, ids.ctypes.data, rows.ctypes.data, 2, 0, None)
    assert k == -3


def test_adam_golden(orc):
    g = np.load(GOLDEN / "adam.npz")
    n, dim = g["w0"].shape
    oa = OrcArena(n, dim, [(int(a), int(b), float(c)) for a, b, c in g["groups"].tolist()], int(g["defer_max"]))
    oa.w[:] = g["w0"]
    for s in range(int(g["steps"])):
        ids = g[f"ids{s}"]
        oa.deferred(ids, g[f"rows{s}"], dim)
        oa.s.step += 0  # step advanced inside
    assert np.array_equal(_bits(oa.w), _bits(g["w"]))
    assert np.array_equal(oa.counter[:n], g["counter"])


# ---- rasterizer (render.hpp:361-640) ---------------------------------------------------------

@pytest.mark.parametrize("seed,n,img,deg", [(5, 4, 16, 2), (11, 8, 24, 3), (400, 6, 32, 3), (401, 6, 32, 1)])
def test_render_forward_backward_bitwise_vs_reference(orc, ref, seed, n, img, deg):
    rows, cam, gt = O.check_scene(seed, n, img, deg)
    geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
    vp = [0, img, 0, img]
    ids = O.ref_cull(geo, cam, vp)
    a = O.render("ref", ids, geo, ng, cam, vp, sh_degree=deg, gt=gt)
    b = O.render("orc", ids, geo, ng, cam, vp, sh_degree=deg, gt=gt)
    for k in ("image", "final_T", "d_img", "rows", "mean2d"):
        assert np.array_equal(_bits(a[k]), _bits(b[k])), k
    assert np.array_equal(a["len"], b["len"])
    assert a["loss"] == b["loss"]


def test_render_synth_scene_split_viewport_bitwise(orc, ref):
    from paper_2509_15645_b200.gss import SynthConfig
    cfg = SynthConfig(n=400, cams=4, width=64, height=48, seed=9, radius_min=2.0, radius_max=3.5, fov_deg=40,
                      fov_ramp=0.8, target_jitter=0.2)
    rows, cams, gts = O.ref_synth(cfg, with_gt=True)
    geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
    for c in range(cfg.cams):
        for vp in ([0, 64, 0, 48], [0, 30, 0, 48], [30, 64, 0, 48]):
            ids = O.ref_cull(geo, cams[c], vp)
            a = O.render("ref", ids, geo, ng, cams[c], vp, gt=gts[c], normalizer=64 * 48 * 3)
            b = O.render("orc", ids, geo, ng, cams[c], vp, gt=gts[c], normalizer=64 * 48 * 3)
            for k in ("image", "final_T", "d_img", "rows", "mean2d"):
                assert np.array_equal(_bits(a[k]), _bits(b[k])), k
            assert a["loss"] == b["loss"]


def test_render_golden(orc):
    g = np.load(GOLDEN / "render.npz")
    b = O.render("orc", g["ids"], g["geo"], g["nongeo"], g["cam"], g["vp"], sh_degree=int(g["deg"]), gt=g["gt"])
    for k in ("image", "d_img", "rows", "mean2d"):
        assert np.array_equal(_bits(b[k]), _bits(g[k])), k
    assert b["loss"] == float(g["loss"])


def test_synth_without_gt_equals_reference_synth_scene(ref):
    """ref_synth_scene_nogt (the reference arm's scene generator at C4 scale, no CPU GT render of all
    views) is pinned to the reference's synth_scene: identical rows and cameras; the GT of a view
    rendered by ref_render_view_rows equals synth_scene's own GT image."""
    import paper_2509_15645_b200 as G

    for seed, n, cams, w, h in ((1, 2000, 5, 48, 40), (7, 500, 3, 32, 32)):
        cfg = G.SynthConfig(seed=seed, n=n, cams=cams, width=w, height=h)
        rows, cam, gts = O.ref_synth(cfg, with_gt=True)
        rows2, cam2 = O.ref_synth_nogt(cfg)
        assert np.array_equal(rows.view(np.uint32), rows2.view(np.uint32))
        assert np.array_equal(cam.view(np.uint32), cam2.view(np.uint32))
        for k in range(cams):
            img = O.ref_render_view(rows2, cam2[k], 3, workers=2)
            assert np.array_equal(img.view(np.uint32), gts[k].view(np.uint32))
