"""Times the host-tier optimizer passes in isolation (no render competing): the forwarding gather
(restore_view with pending grads) and the deferred update on a pinned host arena of N rows with V
visible, staged through HBM (default) or in place (GSS_HOST_STAGING=0). Prints one JSON line."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2509_15645_b200 as G

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40_000_000
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.13
groups = [G.GroupSpec("op", 0, 1, G.Hyperparams(5e-2)), G.GroupSpec("dc", 1, 3, G.Hyperparams(2.5e-3)),
          G.GroupSpec("rest", 4, 45, G.Hyperparams(1.25e-4))]
a = G.Arena(n, 49, groups, 15, interleaved=True, host=True)
a.w.copy_(torch.rand(n, 49))
g = torch.Generator(device="cuda").manual_seed(1)
out = {"n": n, "frac": frac}
t_fp, t_lazy = [], []
for it in range(6):
    ids = torch.nonzero(torch.rand(n, device="cuda", generator=g) < frac).flatten().to(torch.int32)
    rows = torch.randn(ids.numel(), 49, device="cuda")
    pend = G.SparseGrads(ids, rows, 49)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    G.restore_view(a, ids, pend)
    e1.record()
    G.deferred_update(a, pend, want_touched=False, check_invariants=False)
    e2.record()
    torch.cuda.synchronize()
    if it >= 2:
        t_fp.append(e0.elapsed_time(e1))
        t_lazy.append(e1.elapsed_time(e2))
v = float(frac * n)
out.update(fp_ms=float(np.mean(t_fp)), lazy_ms=float(np.mean(t_lazy)),
           fp_gbs=v * 39 * 16 / (np.mean(t_fp) / 1e3) / 1e9)
print(json.dumps(out))
