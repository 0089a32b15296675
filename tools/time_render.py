"""Times rasterize_forward / rasterize_backward per camera on the bench scene (4M Gaussians,
1080p, 8 cameras, training-start parameters vs truth GT) with CUDA events. Used to A/B kernel
variants: GSS_LIB=<variant .so> python tools/time_render.py [N W H reps]. Prints per-camera ms and a
gradient checksum (variants must agree within tolerance)."""
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
import paper_2509_15645_b200 as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1920
H = int(sys.argv[3]) if len(sys.argv) > 3 else 1080
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cfg = bench.scene_config(n, W, H, 8, 1)
truth, cams = G.synth_scene_params(cfg)
td = torch.from_numpy(truth).cuda()
gts = [G.render_view(td, c, 3) for c in cams]
start = torch.from_numpy(bench.training_start(truth)).cuda()
geo = start[:, :10].contiguous()
ng = start[:, 10:].contiguous()
vp = G.viewport_full(W, H)
tf = tb = 0.0
for i, cam in enumerate(cams):
    ids = G.frustum_cull(geo, n, cam, vp)
    sc = G.RenderScene(ids=ids, geo=geo, nongeo=ng)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    fl, bl = [], []
    for r in range(reps + 1):
        ev[0].record()
        fw = G.rasterize_forward(sc, cam, vp, gt=gts[i])
        ev[1].record()
        gb = G.rasterize_backward(sc, cam, fw, fw.d_img)
        ev[2].record()
        torch.cuda.synchronize()
        if r:
            fl.append(ev[0].elapsed_time(ev[1]))
            bl.append(ev[1].elapsed_time(ev[2]))
    fms, bms = float(np.median(fl)), float(np.median(bl))  # median of the timed repetitions
    tf += fms
    tb += bms
    cs = float(gb.rows.double().abs().sum())
    print(f"cam {i}: V {ids.numel():8d} I {fw.instances:9d} fwd {fms:7.3f} ms bwd {bms:7.3f} ms "
          f"loss {float(fw.loss):.6f} |grad| {cs:.6e}")
print(f"total fwd {tf:.3f} ms bwd {tb:.3f} ms (sum over 8 cameras)")
