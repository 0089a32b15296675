"""Generates the golden fixtures in tests/golden/ from the REFERENCE itself (oracle/_ref/libgss_ref.so,
the unmodified reference headers). Run here, where /root/reference exists:

    make -C oracle ref && python tests/golden/make_golden.py

The fixtures travel with the repo so the oracle and the GPU path are pinned even where the
reference cannot be built.
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))
import oracles as O  # noqa: E402

assert O.ref() is not None, "build oracle/_ref/libgss_ref.so first"

# expf on a spread of inputs incl. the two FMA-sensitive points
rng = np.random.default_rng(1)
x = np.concatenate([rng.uniform(-105, 90, 4000), [float.fromhex("0x1.04845ep+5"), -float.fromhex("0x1.f8cbb2p+5"), 0.0, 88.72, -103.97]]).astype(np.float32)
y = np.array([O.ref().ref_expf(float(v)) for v in x], np.float32)
np.savez_compressed(HERE / "expf.npz", x=x, y=y)

# cull: acceptance-5 style scenes + test_render.cpp fixed cases
out = {}
r = O.Rng(77)
k = 0
for _ in range(10):
    rows, cam = O.acceptance5_scene(r)
    vp = np.array([0, 48, 0, 40], np.float32)
    out[f"rows{k}"], out[f"cam{k}"], out[f"vp{k}"], out[f"ids{k}"] = rows, cam, vp, O.ref_cull(rows, cam, vp)
    k += 1
cam = O.basic_cam(64, 64, 60.0, 0.5, 10.0)
rows = np.array([[0, 0, z, -2, -2, -2, 1, 0, 0, 0] for z in (11.0, 0.4, 5.0, -3.0)], np.float32)
vp = np.array([0, 64, 0, 64], np.float32)
out[f"rows{k}"], out[f"cam{k}"], out[f"vp{k}"], out[f"ids{k}"] = rows, cam, vp, O.ref_cull(rows, cam, vp)
k += 1
out["n_cases"] = np.array(k)
np.savez_compressed(HERE / "cull.npz", **out)

# adam: a 20-step sparse schedule with defer_max 15 on a 3-group 49-wide arena
n, dim = 64, 49
groups = np.array([[0, 1, 5e-2], [1, 3, 2.5e-3], [4, 45, 1.25e-4]], np.float64)
ra = O.RefArena(n, dim, [(int(a), int(b), float(c)) for a, b, c in groups], 15)
w0 = rng.uniform(-1, 1, (n, dim)).astype(np.float32)
ra.w[:] = w0
out = dict(w0=w0, groups=groups, defer_max=np.array(15), steps=np.array(20))
for s in range(20):
    ids = np.nonzero(rng.uniform(size=n) < 0.15)[0].astype(np.int32)
    rows = rng.normal(size=(ids.size, dim)).astype(np.float32)
    ra.deferred(ids, rows, dim)
    out[f"ids{s}"], out[f"rows{s}"] = ids, rows
out["w"], out["counter"] = ra.w.copy(), ra.counter.copy()
np.savez_compressed(HERE / "adam.npz", **out)

# render: check scene (test_util.hpp:97-127), forward + L1 + backward
rows, cam, gt = O.check_scene(400, 6, 32, 3)
geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
vp = np.array([0, 32, 0, 32], np.float32)
ids = O.ref_cull(geo, cam, vp)
res = O.render("ref", ids, geo, ng, cam, vp, sh_degree=3, gt=gt)
np.savez_compressed(HERE / "render.npz", ids=ids, geo=geo, nongeo=ng, cam=cam, vp=vp, deg=np.array(3), gt=gt,
                    image=res["image"], d_img=res["d_img"], rows=res["rows"], mean2d=res["mean2d"],
                    loss=np.array(res["loss"], np.float32))
print("golden fixtures written to", HERE)
