import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import paper_2509_15645_b200 as G, bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
cfg = bench.scene_config(n, 1920, 1080, 8, 1)
truth, cams = G.synth_scene_params(cfg)
td = torch.from_numpy(truth).cuda()
gts = np.stack([G.render_view(td, c, 3).cpu().numpy() for c in cams])
del td
e = G.OffloadEngine(bench.training_start(truth), cams, gts)
l, v = e.run(3)
print("visible", v, "loss", l)
