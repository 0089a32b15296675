"""GPU parity of the cull kernel (render.hpp:243-260) through the C ABI: kept ids and the bit
mask must equal the reference bit for bit."""
import numpy as np
import pytest
import torch

import oracles as O
import paper_2509_15645_b200 as G

pytestmark = pytest.mark.gpu


def gpu_cull(rows: np.ndarray, cam_arr: np.ndarray, vp, stride=10, low_pass=0.3):
    geo = torch.from_numpy(np.ascontiguousarray(rows, np.float32).reshape(-1)).cuda()
    n = geo.numel() // stride
    cam = G.camera_from_bytes(cam_arr.tobytes())
    ids, mask = G.frustum_cull(geo, n, cam, G.GssViewport(*map(float, vp)), low_pass, stride=stride, want_mask=True)
    return ids.cpu().numpy(), mask.cpu().numpy().view(np.uint32), n


def mask_from_ids(ids, n):
    words = np.zeros((n + 31) // 32, np.uint64)
    ids = np.asarray(ids, np.int64)
    np.add.at(words, ids // 32, np.left_shift(np.uint64(1), (ids % 32).astype(np.uint64)))
    return words.astype(np.uint32)


def test_expf_device_equals_host_libm(ref):
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(-110, 95, 1 << 20), [float.fromhex("0x1.04845ep+5"), -float.fromhex(
        "0x1.f8cbb2p+5"), 0.0, -0.0, 88.72, 88.73, -103.97, -103.98, np.inf, -np.inf, np.nan]]).astype(np.float32)
    xt = torch.from_numpy(x).cuda()
    yt = torch.empty_like(xt)
    O.ref()  # ensure loaded
    from paper_2509_15645_b200._abi import check, lib
    check(lib().gss_expf_device(xt.data_ptr(), yt.data_ptr(), xt.numel(), torch.cuda.current_stream().cuda_stream))
    y = yt.cpu().numpy()
    sample = np.concatenate([np.arange(0, x.size, 37), np.arange(x.size - 11, x.size)])
    want = np.array([ref.ref_expf(float(v)) for v in x[sample]], np.float32)
    got = y[sample]
    same = (got.view(np.uint32) == want.view(np.uint32)) | (np.isnan(got) & np.isnan(want))
    assert same.all()


def test_depth_plane_exclusions():
    cam = O.basic_cam(64, 64, 60.0, 0.5, 10.0)
    rows = np.array([[0, 0, z, -2, -2, -2, 1, 0, 0, 0] for z in (11.0, 0.4, 5.0, -3.0)], np.float32)
    ids, _, _ = gpu_cull(rows, cam, [0, 64, 0, 64])
    assert list(ids) == [2]


def test_center_always_kept():
    cam = O.basic_cam(32, 32, 40.0)
    rows = np.array([[0, 0, 3, -4, -4, -4, 1, 0, 0, 0]], np.float32)
    ids, _, _ = gpu_cull(rows, cam, [0, 32, 0, 32])
    assert list(ids) == [0]


def test_golden_cases():
    g = np.load(O.ROOT / "tests" / "golden" / "cull.npz")
    for k in range(int(g["n_cases"])):
        ids, _, _ = gpu_cull(g[f"rows{k}"], g[f"cam{k}"], g[f"vp{k}"])
        assert np.array_equal(ids, g[f"ids{k}"]), k


def test_acceptance5_scenes_bit_exact(ref):
    rng = O.Rng(77)
    for _ in range(50):
        rows, cam = O.acceptance5_scene(rng)
        ids, mask, n = gpu_cull(rows, cam, [0, 48, 0, 40])
        want = O.ref_cull(rows, cam, [0, 48, 0, 40])
        assert np.array_equal(ids, want)
        assert np.array_equal(mask, mask_from_ids(want, n))


@pytest.mark.parametrize("n", [1, 31, 511, 512, 513, 1 << 16, 1_000_003])
def test_random_scenes_bit_exact_all_sizes(ref, n):
    rng = np.random.default_rng(n)
    rows = np.zeros((n, 10), np.float32)
    rows[:, 0:3] = rng.uniform(-3, 3, (n, 3))
    rows[:, 3:6] = rng.uniform(-7, 1.0, (n, 3))
    q = rng.normal(size=(n, 4))
    rows[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    cam = O.look_at([0.3, 0.2, -4.0], [0, 0, 0], 300.0, 300.0, 320, 240, 0.5, 8.0)
    for vp in ([0, 320, 0, 240], [0, 160, 0, 240], [160, 320, 0, 240], [-5.5, 20.25, 100, 100.5]):
        ids, mask, _ = gpu_cull(rows, cam, vp)
        want = O.ref_cull(rows, cam, vp)
        assert np.array_equal(ids, want), vp


def test_pathological_rows_bit_exact(ref):
    """NaN/inf/huge values, degenerate quaternions, extreme scales: the fast paths must defer to
    the exact reference predicate."""
    rng = np.random.default_rng(3)
    n = 20000
    rows = np.zeros((n, 10), np.float32)
    rows[:, 0:3] = rng.uniform(-3, 3, (n, 3))
    rows[:, 3:6] = rng.uniform(-10, 10, (n, 3))
    q = rng.normal(size=(n, 4))
    rows[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True)
    specials = np.array([np.nan, np.inf, -np.inf, 1e30, -1e30, 0.0, 1e-30, 88.8, -104.0, 25.0], np.float32)
    for col in range(10):
        idx = rng.choice(n, 300, replace=False)
        rows[idx, col] = rng.choice(specials, 300)
    rows[:50, 6:10] = 0.0
    rows[50:100, 6:10] = 1e-7
    cam = O.look_at([0.0, 0.0, -4.0], [0, 0, 0], 200.0, 200.0, 160, 120, 0.1, 50.0)
    for vp in ([0, 160, 0, 120], [10, 150, 5, 100]):
        ids, _, _ = gpu_cull(rows, cam, vp)
        assert np.array_equal(ids, O.ref_cull(rows, cam, vp))


def test_dense_stride59_arena_bit_exact(ref):
    cfg = G.SynthConfig(n=5000, cams=4, width=64, height=64, seed=2)
    rows, cams, _ = O.ref_synth(cfg)
    for c in cams:
        ids, _, _ = gpu_cull(rows, c, [0, 64, 0, 64], stride=59)
        assert np.array_equal(ids, O.ref_cull(rows, c, [0, 64, 0, 64], stride=59))


def test_synth_c1_scene_bit_exact(ref):
    """The C1 config geometry (100K Gaussians, 256^2) over all 8 cameras."""
    cfg = G.SynthConfig(n=100_000, cams=8, width=256, height=256, seed=1, radius_min=1.5, radius_max=3.0,
                        scale_min=0.003, scale_max=0.01, fov_deg=30)
    rows, cams = G.synth_scene_params(cfg)
    geo = np.ascontiguousarray(rows[:, :10])
    for c in cams:
        ca = O.cam_from_struct(c)
        ids, _, _ = gpu_cull(geo, ca, [0, 256, 0, 256])
        assert np.array_equal(ids, O.ref_cull(geo, ca, [0, 256, 0, 256]))


@pytest.mark.parametrize("seed", range(6))
def test_border_stress_bit_exact(ref, seed):
    """Centres placed within a few ulps..pixels of the viewport borders (where the fast
    classifier's error margins decide), scales spanning the radius bound, random cameras
    including non-orthonormal rotations and low-pass values 0 / 0.3 / 10."""
    rng = np.random.default_rng(100 + seed)
    n = 200_000
    W_, H_ = 640, 360
    cam = O.look_at(list(rng.uniform(-3, 3, 3)), list(rng.uniform(-0.5, 0.5, 3)), float(rng.uniform(200, 900)),
                    float(rng.uniform(200, 900)), W_, H_, 0.05, 30.0)
    if seed % 2 == 1:  # perturb the rotation (no longer orthonormal)
        cam = cam.copy()
        cam[:9] = cam[:9] * rng.uniform(0.7, 1.3, 9).astype(np.float32)
    rot = cam[:9].reshape(3, 3).astype(np.float64)
    t = cam[9:12].astype(np.float64)
    fx, fy, cx, cy = [float(v) for v in cam[12:16]]
    # sample pixel targets near the borders, then back-project at random depths
    u = np.where(rng.random(n) < 0.5, rng.choice([0.0, W_], n) + rng.normal(0, 3, n), rng.uniform(-50, W_ + 50, n))
    v = np.where(rng.random(n) < 0.5, rng.choice([0.0, H_], n) + rng.normal(0, 3, n), rng.uniform(-50, H_ + 50, n))
    z = rng.uniform(0.1, 20.0, n)
    pc = np.stack([(u - cx) / fx * z, (v - cy) / fy * z, z], 1)
    pw = np.linalg.solve(rot, (pc - t).T).T
    rows = np.zeros((n, 10), np.float32)
    rows[:, 0:3] = pw
    rows[:, 3:6] = rng.uniform(-9, -1, (n, 3))
    q = rng.normal(size=(n, 4))
    rows[:, 6:10] = q / np.linalg.norm(q, axis=1, keepdims=True) * rng.choice([1.0, 1e-13, 7.0], (n, 1))
    for lp in (0.3, 0.0, 10.0):
        for vp in ([0, W_, 0, H_], [0.25, W_ - 0.5, 1.0, H_ * 0.5]):
            ids, mask, _ = gpu_cull(rows, cam, vp, low_pass=lp)
            want = O.ref_cull(rows, cam, vp, low_pass=lp)
            assert np.array_equal(ids, want), (lp, vp, np.setxor1d(ids, want)[:10])
            assert np.array_equal(mask, mask_from_ids(want, n))
