import sys, types
sys.path.insert(0, '/root/repo')
import torch, numpy as np
import paper_2509_15645_b200 as G, bench
a = types.SimpleNamespace(n=4_000_000, width=1920, height=1080, cams=8, seed=1)
cfg = bench.scene_config(a.n, a.width, a.height, a.cams, a.seed)
truth, cams = G.synth_scene_params(cfg)
res = bench.kernel_probe(G, truth, cams, torch.device('cuda', 0), a)
for r in res: print(r)
