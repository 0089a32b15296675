import sys, numpy as np
sys.path.insert(0,'/root/repo'); sys.path.insert(0,'/root/repo/tests')
import paper_2509_15645_b200 as G, bench
for cams in (8, 1):
    cfg=bench.scene_config(4_000_000,1920,1080,cams,1)
    rows,cs=G.synth_scene_params(cfg)
    with open(f'/root/repo/paper_2509_15645_b200/_build/cull_c{cams}.bin','wb') as f:
        f.write(np.int64(rows.shape[0]).tobytes()); f.write(bytes(cs[0])); f.write(np.ascontiguousarray(rows[:,:10]).tobytes())
