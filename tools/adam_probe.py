"""Isolated HBM optimizer passes at C4 scale on the engine's layout (row-interleaved 49-wide
non-geometric arena, defer_max 15; 10-wide geometric arena, defer_max 0): deferred update,
forwarding gather (restore_view with pending grads) and dense geo update, each timed with CUDA
events over repeated launches after the counters reach steady state. Algorithmic bytes as
SURVEY.md §8d. GSS_LIB=<variant .so> selects a build variant. Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2509_15645_b200 as G  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40_000_000
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1292
peak = 6543.4
opt = G.OptimConfig()
ng = G.Arena(n, 49, opt.nongeo_groups(), 15, interleaved=True)
geo = G.Arena(n, 10, opt.geo_groups(), 0)
gen = torch.Generator(device="cuda").manual_seed(7)
ng.w.copy_(torch.rand(n, 49, device="cuda", generator=gen) * 2 - 1)
geo.w.copy_(torch.rand(n, 10, device="cuda", generator=gen) * 2 - 1)


def draw():  # gradient rows in the engine's stage layouts: non-geometric 52-float rows, geometric 10
    ids = torch.nonzero(torch.rand(n, device="cuda", generator=gen) < frac).flatten().to(torch.int32)
    return ids, torch.randn(ids.numel(), 52, device="cuda", generator=gen), torch.randn(ids.numel(), 10, device="cuda",
                                                                                          generator=gen)


sets = [draw() for _ in range(4)]
for it in range(20):  # steady-state counters
    ids, rows, _ = sets[it % 4]
    G.deferred_update(ng, G.SparseGrads(ids, rows, 52, 0), want_touched=False, check_invariants=False)
torch.cuda.synchronize()
res = {"n": n, "frac": frac, "lib": os.environ.get("GSS_LIB", "default")}
reps = 8
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
# deferred update (touched count read back for the byte count)
tms, tbytes = [], []
for r in range(reps):
    ids, rows, _ = sets[r % 4]
    ev[0].record()
    t = G.deferred_update(ng, G.SparseGrads(ids, rows, 52, 0), want_touched=False, check_invariants=False)
    ev[1].record()
    torch.cuda.synchronize()
    touched = int(t.item())
    tms.append(ev[0].elapsed_time(ev[1]))
    tbytes.append(touched * 4 * 49 * 6 + ids.numel() * 4 * 49 + 2 * n)
res["deferred_ms"] = float(np.median(tms))
res["deferred_frac"] = float(np.median(tbytes)) / (res["deferred_ms"] / 1e3) / 1e9 / peak
# forwarding gather with pending grads
ids, rows, _ = sets[0]
pids, prow, _ = sets[1]
pend = G.SparseGrads(pids, prow, 52, 0)
out = torch.empty(ids.numel(), 49, device="cuda")
gms = []
for r in range(reps):
    ev[0].record()
    G.restore_view(ng, ids, pend, out=out)
    ev[1].record()
    torch.cuda.synchronize()
    gms.append(ev[0].elapsed_time(ev[1]))
V, Vp = ids.numel(), pids.numel()
res["gather_ms"] = float(np.median(gms))
res["gather_frac"] = (V * (3 * 196 + 1) + Vp * 196 + V * 196) / (res["gather_ms"] / 1e3) / 1e9 / peak
# dense geo update (defer_max 0)
dms = []
for r in range(reps):
    ids, _, grows = sets[r % 4]
    ev[0].record()
    G.deferred_update(geo, G.SparseGrads(ids, grows, 10, 0), want_touched=False, check_invariants=False)
    ev[1].record()
    torch.cuda.synchronize()
    dms.append(ev[0].elapsed_time(ev[1]))
res["geo_ms"] = float(np.median(dms))
res["geo_frac"] = (240 * n + 40 * sets[0][0].numel()) / (res["geo_ms"] / 1e3) / 1e9 / peak
print(json.dumps(res))
