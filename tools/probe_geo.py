"""Isolated dense geo Adam pass (engine.hpp:380-386 at 4M Gaussians, 8.28% sparse grads): the
command profiled by ncu for update_kernel<16,0,1>. Prints the CUDA-event time per call."""
import ctypes as C
import sys

import torch

sys.path.insert(0, "/root/repo")
import paper_2509_15645_b200 as G  # noqa: E402
from paper_2509_15645_b200._abi import check, lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dev = torch.device("cuda", 0)
opt = G.OptimConfig()
gen = torch.Generator(device=dev)
gen.manual_seed(7)
ar = G.Arena(n, 10, opt.geo_groups(), 0, device=dev)
ar.w.uniform_(-1, 1)
gi = torch.nonzero(torch.rand(n, device=dev, generator=gen) < 0.0828).flatten().to(torch.int32)
gg = torch.randn(gi.numel(), 10, device=dev, generator=gen)
st = ar.c_struct()
gs = G.SparseGrads(gi, gg, 10).c_struct()
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    check(lib().gss_deferred_update(C.byref(st), C.byref(gs), None, None, s))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda._sleep(20_000_000)
e0.record()
for _ in range(reps):
    check(lib().gss_deferred_update(C.byref(st), C.byref(gs), None, None, s))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
b = 240 * n + 44 * gi.numel()
print(f"geo dense update: {ms * 1e3:.1f} us, {b / ms / 1e6:.0f} GB/s algorithmic")
