"""GPU parity of the rasterizer (render.hpp:361-640) through the C ABI.

Forward: image, final transmittance and per-pixel used-contribution counts are bit-identical to
the reference (same splat order, same membership, same op sequence, glibc-exact expf).
Loss: identical L1 value and gradient image. Backward: the reference accumulates per-slot sums
in pixel order, the device in per-tile trees (deterministic, different association) and recovers
transmittance by division, so gradients match within the stated fp32 tolerance:
    rel_err (test_util.hpp:17-19) <= 1e-4 on every entry  (the north-star contract), and
    rel_err_floor with floor 1e-3 * max|g| <= 2e-3        (a scale-aware check that catches bugs).
"""
import numpy as np
import pytest
import torch

import oracles as O
import paper_2509_15645_b200 as G

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def gpu_render(ids, geo, ng, cam_arr, vp, *, deg=3, bg=(0, 0, 0), gt=None, normalizer=0, compact=False,
               d_img=None):
    geo_t = torch.from_numpy(np.ascontiguousarray(geo, np.float32)).cuda()
    ng_t = torch.from_numpy(np.ascontiguousarray(ng, np.float32)).cuda()
    ids_t = torch.from_numpy(np.ascontiguousarray(ids, np.int32)).cuda()
    cam = G.camera_from_bytes(cam_arr.tobytes())
    sc = G.RenderScene(ids=ids_t, geo=geo_t, nongeo=ng_t, nongeo_compact=compact, sh_degree=deg, background=bg)
    gt_t = None if gt is None else torch.from_numpy(np.ascontiguousarray(gt, np.float32)).cuda()
    rr = G.rasterize_forward(sc, cam, G.GssViewport(*map(float, vp)), gt=gt_t, normalizer=normalizer)
    dimg = rr.d_img if d_img is None else torch.from_numpy(np.ascontiguousarray(d_img, np.float32)).cuda()
    gb = G.rasterize_backward(sc, cam, rr, dimg if dimg is not None else torch.zeros_like(rr.image))
    torch.cuda.synchronize()
    return dict(image=rr.image.cpu().numpy(), final_T=rr.final_T.cpu().numpy(), len=rr.n_contrib.cpu().numpy(),
                loss=None if rr.loss is None else float(rr.loss.item()),
                d_img=None if rr.d_img is None else rr.d_img.cpu().numpy(), rows=gb.rows.cpu().numpy(),
                mean2d=gb.mean2d.cpu().numpy(), instances=rr.instances)


def grad_metrics(a, b):
    g = np.abs(a).max() if a.size else 0.0
    floor = max(1e-12, 1e-3 * g)
    return float(O.rel_err(a, b).max(initial=0.0)), float(O.rel_err_floor(a, b, floor).max(initial=0.0))


def check_parity(r, g, *, loss=True):
    assert np.array_equal(bits(r["image"]), bits(g["image"]))
    assert np.array_equal(bits(r["final_T"]), bits(g["final_T"]))
    assert np.array_equal(r["len"], g["len"])
    if loss:
        assert r["loss"] == g["loss"]
        assert np.array_equal(bits(r["d_img"]), bits(g["d_img"]))
    for k in ("rows", "mean2d"):
        rel, relf = grad_metrics(r[k], g[k])
        print(f"{k}: rel_err {rel:.3e} rel_err_floor {relf:.3e}")
        assert rel <= 1e-4, k
        assert relf <= 2e-3, k


@pytest.mark.parametrize("seed,n,img,deg", [(5, 4, 16, 2), (11, 8, 24, 3), (400, 6, 32, 3), (401, 6, 32, 0),
                                            (402, 40, 48, 3)])
def test_check_scenes(ref, seed, n, img, deg):
    rows, cam, gt = O.check_scene(seed, n, img, deg)
    geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
    vp = [0, img, 0, img]
    ids = O.ref_cull(geo, cam, vp)
    r = O.render("ref", ids, geo, ng, cam, vp, sh_degree=deg, gt=gt)
    g = gpu_render(ids, geo, ng, cam, vp, deg=deg, gt=gt)
    check_parity(r, g)


def test_golden_fixture():
    gg = np.load(O.ROOT / "tests" / "golden" / "render.npz")
    g = gpu_render(gg["ids"], gg["geo"], gg["nongeo"], gg["cam"], gg["vp"], deg=int(gg["deg"]), gt=gg["gt"])
    assert np.array_equal(bits(g["image"]), bits(gg["image"]))
    assert np.array_equal(bits(g["d_img"]), bits(gg["d_img"]))
    assert g["loss"] == float(gg["loss"])
    rel, relf = grad_metrics(gg["rows"], g["rows"])
    assert rel <= 1e-4 and relf <= 2e-3


def test_zero_gaussians_render_background():
    cam = O.basic_cam(8, 8, 10.0)
    for bg in ((0, 0, 0), (1, 1, 1)):
        g = gpu_render(np.zeros(0, np.int32), np.zeros((1, 10), np.float32), np.zeros((1, 49), np.float32), cam,
                       [0, 8, 0, 8], bg=bg)
        assert np.all(g["image"] == bg[0])


def test_saturated_gaussian_center(ref):
    """test_render.cpp:245-264: alpha clamps at 0.999."""
    geo = np.array([[0, 0, 1, np.log(0.5), np.log(0.5), np.log(0.5), 1, 0, 0, 0]], np.float32)
    ng = np.zeros((1, 49), np.float32)
    ng[0, 0] = 20.0
    ng[0, 1] = (1.0 - 0.5) / 0.28209479177387814
    ng[0, 2] = (0.0 - 0.5) / 0.28209479177387814
    ng[0, 3] = (0.0 - 0.5) / 0.28209479177387814
    cam = O.basic_cam(9, 9, 10.0)
    g = gpu_render(np.array([0], np.int32), geo, ng, cam, [0, 9, 0, 9], deg=0)
    r = O.render("ref", [0], geo, ng, cam, [0, 9, 0, 9], sh_degree=0)
    assert np.array_equal(bits(g["image"]), bits(r["image"]))
    assert abs(g["image"][4, 4, 0] - 0.999) < 1e-6


def test_depth_ties_break_by_ascending_id(ref):
    """test_render.cpp:308-332."""
    geo = np.array([[-0.01, 0, 1.5] + [np.log(0.4)] * 3 + [1, 0, 0, 0],
                    [0.01, 0, 1.5] + [np.log(0.4)] * 3 + [1, 0, 0, 0]], np.float32)
    ng = np.zeros((2, 49), np.float32)
    ng[:, 0] = 0.0
    ng[0, 1] = (1.0 - 0.5) / 0.28209479177387814
    ng[1, 2] = (1.0 - 0.5) / 0.28209479177387814
    cam = O.basic_cam(7, 7, 10.0)
    g = gpu_render(np.array([0, 1], np.int32), geo, ng, cam, [0, 7, 0, 7], deg=0)
    r = O.render("ref", [0, 1], geo, ng, cam, [0, 7, 0, 7], sh_degree=0)
    assert np.array_equal(bits(g["image"]), bits(r["image"]))
    assert g["len"][3, 3] == 2


def test_zero_image_gradient_gives_exact_zero_grads():
    rows, cam, gt = O.check_scene(5, 4, 16, 2)
    geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
    ids = O.ref_cull(geo, cam, [0, 16, 0, 16])
    g = gpu_render(ids, geo, ng, cam, [0, 16, 0, 16], deg=2, d_img=np.zeros((16, 16, 3), np.float32))
    assert np.all(g["rows"] == 0)


def test_occluded_gaussian_gradient_small(ref):
    """test_render.cpp:397-428 (double there; float here): occluded grads <= ~1e-3 of the occluder."""
    geo = np.array([[0, 0, 1] + [np.log(4.0)] * 3 + [1, 0, 0, 0], [0, 0, 1.5] + [np.log(6.0)] * 3 + [1, 0, 0, 0]],
                   np.float32)
    ng = np.zeros((2, 49), np.float32)
    ng[:, 0] = 20.0
    ng[:, 1] = (0.8 - 0.5) / 0.28209479177387814
    cam = O.basic_cam(5, 5, 50.0)
    d = np.random.default_rng(9).uniform(-1, 1, (5, 5, 3)).astype(np.float32)
    g = gpu_render(np.array([0, 1], np.int32), geo, ng, cam, [0, 5, 0, 5], deg=0, d_img=d)
    nf, nb = np.abs(g["rows"][0]).max(), np.abs(g["rows"][1]).max()
    assert nf > 0 and nb <= 1.0001e-3 * nf


def test_determinism_bitwise_across_runs():
    rows, cam, gt = O.check_scene(11, 8, 24, 3)
    geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
    ids = O.ref_cull(geo, cam, [0, 24, 0, 24])
    a = gpu_render(ids, geo, ng, cam, [0, 24, 0, 24], gt=gt)
    b = gpu_render(ids, geo, ng, cam, [0, 24, 0, 24], gt=gt)
    for k in ("image", "rows", "mean2d"):
        assert np.array_equal(bits(a[k]), bits(b[k]))


@pytest.mark.parametrize("vp", [[0, 64, 0, 48], [0, 30, 0, 48], [30, 64, 0, 48], [7.3, 50.6, 3.2, 40.1]])
def test_synth_scene_split_viewports(ref, vp):
    cfg = G.SynthConfig(n=400, cams=3, width=64, height=48, seed=9, radius_min=2.0, radius_max=3.5, fov_deg=40,
                        fov_ramp=0.8, target_jitter=0.2)
    rows, cams, gts = O.ref_synth(cfg, with_gt=True)
    geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
    for c in range(cfg.cams):
        ids = O.ref_cull(geo, cams[c], vp)
        r = O.render("ref", ids, geo, ng, cams[c], vp, gt=gts[c], normalizer=64 * 48 * 3)
        g = gpu_render(ids, geo, ng, cams[c], vp, gt=gts[c], normalizer=64 * 48 * 3)
        check_parity(r, g)


def test_compact_nongeo_rows(ref):
    cfg = G.SynthConfig(n=300, cams=2, width=40, height=40, seed=3)
    rows, cams, gts = O.ref_synth(cfg, with_gt=True)
    geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
    ids = O.ref_cull(geo, cams[0], [0, 40, 0, 40])
    r = O.render("ref", ids, geo, ng[ids], cams[0], [0, 40, 0, 40], compact=True, gt=gts[0])
    g = gpu_render(ids, geo, ng[ids], cams[0], [0, 40, 0, 40], compact=True, gt=gts[0])
    check_parity(r, g)


def test_c1_scene_256(ref):
    """C1 geometry (100K, 256^2) for one camera: forward bit-exact; grads in tolerance."""
    cfg = G.SynthConfig(n=100_000, cams=8, width=256, height=256, seed=1, radius_min=1.5, radius_max=3.0,
                        scale_min=0.003, scale_max=0.01, fov_deg=30)
    rows, cams = G.synth_scene_params(cfg)
    geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
    cam = O.cam_from_struct(cams[0])
    ids = O.ref_cull(geo, cam, [0, 256, 0, 256])
    gt = np.random.default_rng(0).uniform(0, 1, (256, 256, 3)).astype(np.float32)
    r = O.render("ref", ids, geo, ng, cam, [0, 256, 0, 256], gt=gt)
    g = gpu_render(ids, geo, ng, cam, [0, 256, 0, 256], gt=gt)
    print("visible", ids.size, "contribs", r["contribs"], "instances", g["instances"])
    check_parity(r, g)


@pytest.mark.parametrize("seed", [3, 17])
def test_forward_adversarial_geometry_bit_exact(ref, seed):
    """Edge geometry for the composite's exact quotient and expf: needle-like splats (one log-scale
    at -9..-6, condition numbers far beyond any per-record range certificate), huge splats covering
    the whole view, and means placed on pixel centres by inverse projection (numerators of the
    conic form near or exactly zero). Image, final T, counts and loss stay bit-identical to the
    reference renderer; gradients within the tolerance."""
    rng = np.random.default_rng(seed)
    W, H = 40, 32
    cam = O.look_at([0.2, -0.1, -3.0], [0.0, 0.0, 0.0], 60.0, 55.0, W, H, 0.1, 50.0)
    R = cam[0:9].astype(np.float64).reshape(3, 3)
    t = cam[9:12].astype(np.float64)
    fx, fy, cx, cy = (float(v) for v in cam[12:16])
    n = 240
    rows = np.zeros((n, 59), np.float32)
    for i in range(n):
        if i % 3 == 0:  # mean on a pixel centre at a random depth
            u, v, z = rng.integers(0, W) + 0.5, rng.integers(0, H) + 0.5, rng.uniform(2.0, 4.0)
            pc = np.array([(u - cx) / fx * z, (v - cy) / fy * z, z])
            rows[i, 0:3] = R.T @ (pc - t)
        else:
            rows[i, 0:3] = rng.uniform(-0.6, 0.6, 3)
        kind = i % 4
        if kind == 0:
            ls = [rng.uniform(-9, -6), rng.uniform(-3, -1), rng.uniform(-3, -1)]  # needle
        elif kind == 1:
            ls = [rng.uniform(-1.0, 0.5)] * 3  # huge: covers the view
        else:
            ls = rng.uniform(-4.5, -2.0, 3)
        rows[i, 3:6] = rng.permutation(ls)
        q = rng.normal(size=4)
        rows[i, 6:10] = q / np.linalg.norm(q)
        rows[i, 10] = rng.uniform(-3.0, 1.0)
        rows[i, 11:14] = rng.uniform(-1.0, 1.0, 3)
        rows[i, 14:] = rng.normal(0, 0.1, 45)
    geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
    vp = [0, W, 0, H]
    ids = O.ref_cull(geo, cam, vp)
    assert ids.size > 100
    gt = rng.uniform(0, 1, (H, W, 3)).astype(np.float32)
    r = O.render("ref", ids, geo, ng, cam, vp, gt=gt)
    g = gpu_render(ids, geo, ng, cam, vp, gt=gt)
    check_parity(r, g)
