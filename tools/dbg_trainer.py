import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2509_15645_b200 as G
from paper_2509_15645_b200 import imgpar as IP
from test_imgpar_gpu import scene
rows, cams, gts = scene(13, 4000, 80, 64)
K = 4
for rep in range(2):
    tr = IP.ShardTrainer(rows, cams, gts)
    print("trainer", [tr.step() for _ in range(K)])
gh = np.stack([g.cpu().numpy() for g in gts])
for pipe in (False, True):
    eng = G.OffloadEngine(rows, cams, gh, pipelined=pipe)
    print("engine", pipe, eng.run(K)[0].tolist())
    eng.close()
# manual: engine-like serial using gss API directly with rasterize_forward/backward (no split phase)
opt = G.OptimConfig()
dev = torch.device("cuda")
r = torch.from_numpy(rows).cuda()
geo = G.Arena(rows.shape[0], 10, opt.geo_groups(), 0, device=dev); geo.w.copy_(r[:, :10])
ng = G.Arena(rows.shape[0], 49, opt.nongeo_groups(), 15, device=dev); ng.w.copy_(r[:, 10:])
pending = None; out = []
for g in range(K):
    cam = cams[g % 4]; vp = G.viewport_full(cam.width, cam.height)
    ids = G.frustum_cull(geo.w, geo.count, cam, vp)
    fwd = G.restore_view(ng, ids, pending)
    if pending is not None:
        G.deferred_update(ng, pending, want_touched=False, check_invariants=False)
    sc = G.RenderScene(ids=ids, geo=geo.w, nongeo=fwd, nongeo_compact=True)
    fw = G.rasterize_forward(sc, cam, vp, gt=gts[g % 4])
    gb = G.rasterize_backward(sc, cam, fw, fw.d_img)
    out.append(float(fw.loss.item()))
    G.deferred_update(geo, G.SparseGrads(ids, gb.rows, 59, 0), want_touched=False, check_invariants=False)
    pending = G.SparseGrads(ids, gb.rows, 59, 10)
print("manual", out)
