"""Rasterizer work accounting on the bench scene: for each camera, the forward / backward useful
fraction (contributions composited / lane-pixel slots the kernels offered) and the average
contributions per pixel, from a library built with -DGSS_RASTER_STATS=1:

  python -c "from paper_2509_15645_b200 import build; build.build_lib(variant='stats', defines=('GSS_RASTER_STATS=1',))"
  GSS_LIB=paper_2509_15645_b200/_build/var_stats/libgss_b200.so python tools/raster_work.py N W H [out.json]

Timing in this run is not representative (counters use atomics); CUDA-event times come from the
product library (tools/time_render.py)."""
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import bench  # noqa: E402
import paper_2509_15645_b200 as G  # noqa: E402
from paper_2509_15645_b200._abi import lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1920
H = int(sys.argv[3]) if len(sys.argv) > 3 else 1080
assert lib().gss_raster_stats_enabled() == 1, "load the GSS_RASTER_STATS=1 variant through GSS_LIB"
truth, cams = G.synth_scene_params(bench.scene_config(n, W, H, 8, 1))
td = torch.from_numpy(truth).cuda()
gts = [G.render_view(td, c, 3) for c in cams]
del td
start = torch.from_numpy(bench.training_start(truth)).cuda()
geo, ng = start[:, :10].contiguous(), start[:, 10:].contiguous()
vp = G.viewport_full(W, H)
buf = (C.c_uint64 * 8)()
rows = []
tot = np.zeros(8)
for i, cam in enumerate(cams):
    ids = G.frustum_cull(geo, n, cam, vp)
    sc = G.RenderScene(ids=ids, geo=geo, nongeo=ng)
    lib().gss_raster_stats(buf, 1)
    fw = G.rasterize_forward(sc, cam, vp, gt=gts[i])
    G.rasterize_backward(sc, cam, fw, fw.d_img)
    lib().gss_raster_stats(buf, 1)
    s = np.array(list(buf), np.float64)
    tot += s
    r = {"cam": i, "visible": int(ids.numel()), "instances": int(fw.instances),
         "fwd_in_box_per_px": s[2] / (W * H), "fwd_composited_per_px": s[3] / (W * H),
         "fwd_useful_of_offered": s[3] / max(s[1], 1), "fwd_useful_of_eval_slots": s[3] / max(s[4], 1),
         "bwd_useful_per_px": s[7] / (W * H), "bwd_useful_of_offered": s[7] / max(s[6], 1)}
    rows.append(r)
    print(json.dumps(r))
summary = {"n": n, "width": W, "height": H,
           "fwd_composited_per_px": tot[3] / (8 * W * H), "fwd_useful_of_offered": tot[3] / tot[1],
           "fwd_useful_of_eval_slots": tot[3] / tot[4], "fwd_in_box_per_px": tot[2] / (8 * W * H),
           "bwd_useful_per_px": tot[7] / (8 * W * H), "bwd_useful_of_offered": tot[7] / tot[6],
           "cams": rows}
print(json.dumps({k: v for k, v in summary.items() if k != "cams"}))
if len(sys.argv) > 4:
    json.dump(summary, open(sys.argv[4], "w"), indent=1)
