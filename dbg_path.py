import sys, numpy as np
sys.path.insert(0,'/root/repo/tests'); sys.path.insert(0,'/root/repo')
import oracles as O
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
np.save('/tmp/dbg/rows.npy', rows); np.save('/tmp/dbg/cam.npy', cam)
for vp in ([0, 160, 0, 120], [10, 150, 5, 100]):
    a = O.ref_cull(rows, cam, vp); b = O.orc_cull(rows, cam, vp)
    print(len(a), len(b), np.setxor1d(a,b)[:20])
    if len(sys.argv)>1:
        import torch, paper_2509_15645_b200 as G
        geo = torch.from_numpy(rows.reshape(-1).copy()).cuda()
        ids, m = G.frustum_cull(geo, n, G.camera_from_bytes(cam.tobytes()), G.GssViewport(*map(float, vp)), 0.3, stride=10, want_mask=True)
        g = ids.cpu().numpy()
        d = np.setxor1d(a, g)
        print("gpu", len(g), "diff", len(d))
        for i in d[:40]:
            print(i, i in a, i in g, rows[i].tolist())
