import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch
import paper_2509_15645_b200 as G
import oracles as O
for n in (100_000, 4_000_000):
    dim, dens, passes = 49, 0.0828, 100
    grp = [G.GroupSpec("all", 0, dim, G.Hyperparams(1e-3))]
    gen = torch.Generator(device="cuda"); gen.manual_seed(7)
    dense = G.Arena(n, dim, grp, 0)
    d1 = G.Arena(n, dim, grp, 15, interleaved=True)
    d2 = G.Arena(n, dim, grp, 15, interleaved=False)
    w0 = torch.rand((n, dim), device="cuda", generator=gen) * 2 - 1
    for a in (dense, d1, d2): a.w.copy_(w0)
    for p in range(passes):
        ids = torch.nonzero(torch.rand(n, device="cuda", generator=gen) < dens).flatten().to(torch.int32)
        rows = torch.randn(ids.numel(), dim, device="cuda", generator=gen)
        g = torch.zeros((n, dim), device="cuda"); g[ids.long()] = rows
        G.adam_step_dense(dense, g)
        for a in (d1, d2): G.deferred_update(a, G.SparseGrads(ids, rows, dim), want_touched=False)
    for a in (d1, d2): G.flush_deferred(a)
    e1 = O.rel_err(dense.w.cpu().numpy(), d1.w.cpu().numpy())
    e2 = O.rel_err(dense.w.cpu().numpy(), d2.w.cpu().numpy())
    same = torch.equal(d1.w, d2.w)
    i = np.unravel_index(np.argmax(e1), e1.shape)
    print(n, "dev interleaved", e1.max(), "separate", e2.max(), "identical", same, "argmax", i,
          "counter", int(d1.counter[i[0]]), "w", float(dense.w[i]), float(d1.w[i]), "v", float(dense.v[i]), float(d1.v[i]))
