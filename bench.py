"""bench.py — GS-Scale per-iteration training step on the B200.

Workload (BASELINE.json configs[3], "C4" of SURVEY.md §8, the largest single-GPU configuration):
a synthetic 40M-Gaussian scene (the reference generator, synth.hpp:100-159, scales shrunk by
(1e5/N)^(1/3) so depth complexity stays bounded), 3840x2160 views, selective offload (geometric
tier always in HBM; the non-geometric tier placed by the HBM budget — in HBM when it fits, the
north_star's "or from HBM when the scene fits in 180 GB", else pinned host memory), pipelined
two-stream engine, deferred Adam (defer_max = 15) for the non-geometric tier, dense immediate Adam
for the geometric tier. The same scene with the non-geometric tier forced to pinned host memory is
reported under `host_offload`. A step = one OffloadEngine iteration: cull(g) + forwarding gather
(restore_view + pending pass) + rasterize forward + L1 loss + rasterize backward + geo Adam +
handoff + lazy deferred Adam(g-1).

Arms:
  default            our sm_100a path (libgss_b200.so through its C ABI);
  --impl reference   the reference's own CPU implementation (oracle/_ref/libgss_ref.so: the
                     unmodified reference headers compiled on this host) on the same workload, all
                     host threads. The reference renderer cannot render a C4 view (its per-pixel
                     CSR offsets are int32, render.hpp:273, and a 3840x2160 view here has ~3.7e9
                     contributions), so each reference step is a bounded sample of the iteration:
                     its O(N) stages at full size and the rasterizer on sub-viewports, extrapolated
                     to the full view (see ref_stage_sample).

One JSON line on rank 0. Timing: W untimed warm-up iterations, then K iterations bracketed by
barrier + device sync, CUDA events on the launching streams; inputs (30 GB of w/m/v state at C4)
are far larger than the 126 MB L2, so no flush is needed between iterations.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "training iters/sec & Gaussians culled/s at N Gaussians; Adam/cull HBM GB/s vs peak"
FALLBACK_HBM_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--gaussians", "--n", dest="n", type=int, default=40_000_000)
    p.add_argument("--width", type=int, default=3840)
    p.add_argument("--height", type=int, default=2160)
    p.add_argument("--cams", type=int, default=8)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--nongeo-on-host", action="store_true",
                   help="force the non-geometric tier (w/m/v) into pinned host memory (= --nongeo-tier host)")
    p.add_argument("--nongeo-tier", default="auto", choices=["auto", "hbm", "host"],
                   help="selective offload: placement of the non-geometric tier (auto: HBM when it fits the budget)")
    p.add_argument("--no-host-offload", action="store_true",
                   help="skip the extra run with the non-geometric tier forced to pinned host memory")
    p.add_argument("--no-probe", action="store_true", help="skip the isolated HBM kernel probe")
    p.add_argument("--mode", default="auto", choices=["auto", "engine", "imgpar", "replicas"],
                   help="auto: the two-stream engine at N=1, image-parallel sharded training at N>1; "
                        "imgpar: sharded training with image-parallel rendering (any N); "
                        "replicas: N independent engines (weak-scaling replicas, no collective)")
    p.add_argument("--ref-max-steps", type=int, default=2,
                   help="reference arm: cap on timed CPU sample steps (each is ~30 s at the default workload)")
    return p.parse_args()


def scene_config(n, w, h, cams, seed):
    """C1's SynthConfig scaled to n Gaussians and a w x h view."""
    import paper_2509_15645_b200 as G

    s = (1e5 / n) ** (1.0 / 3.0)
    return G.SynthConfig(seed=seed, n=n, cams=cams, width=w, height=h, radius_min=1.5, radius_max=3.0,
                         scale_min=0.003 * s, scale_max=0.01 * s, fov_deg=30.0)


def training_start(truth: np.ndarray) -> np.ndarray:
    """Truth with opacity logit(0.1) and SH bands >= 1 zeroed."""
    start = truth.copy()
    start[:, 10] = np.float32(np.log(0.1 / 0.9))
    start[:, 14:] = 0.0
    return start


class Clocks:
    """SM clock / throttle-reason sampler running only during the timed region: NVML polled every
    5 ms from a thread (the timed regions are ~0.1 s, too short for nvidia-smi's process start and
    100 ms period), with nvidia-smi as the fallback when NVML is unavailable."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NVML_REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.p = self.t = None
        self.samples, self.reasons, self.mx = [], set(), 0.0
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                ent = vis.split(",")[index].strip()
                h = nv.nvmlDeviceGetHandleByUUID(ent) if ent.startswith("GPU-") else nv.nvmlDeviceGetHandleByIndex(int(ent))
            else:
                h = nv.nvmlDeviceGetHandleByIndex(index)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.stop_ev = threading.Event()
            first = threading.Event()

            def run():
                while not self.stop_ev.is_set():
                    self.samples.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for nm, bit in self.NVML_REASONS.items():
                        if r & bit:
                            self.reasons.add(nm)
                    first.set()
                    time.sleep(0.005)

            self.t = threading.Thread(target=run, daemon=True)
            self.t.start()
            first.wait(1.0)
            return
        except Exception:
            self.t = None
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                      stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.t is not None:
            self.stop_ev.set()
            self.t.join()
            if not self.samples:
                return None
            return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.mx,
                    "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}
        if self.p is None:
            return None
        self.p.terminate()
        self.p.wait()
        self.f.seek(0)
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.f.read().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.f.name)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvidia-smi"}


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            d = json.loads(f.read_text())
            for k in ("hbm_gbs", "hbm_GBs", "hbm"):
                if k in d:
                    v = d[k]
                    return float(v["burst"] if isinstance(v, dict) else v), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


# ---------------------------------------------------------------------------------------------

def tier_placement(a, n, dev) -> str:
    """Selective offload (store.hpp:149-192): the geometric tier always lives in HBM; the
    non-geometric tier (640 B/row interleaved w/m/v + counter) goes to HBM when it fits beside the
    geometric tier, the per-iteration staging (sized for the whole scene) and the rasterizer with
    a 25% margin, else to pinned host memory."""
    if a.nongeo_on_host:
        return "host"
    if a.nongeo_tier != "auto":
        return a.nongeo_tier
    import torch

    free, _ = torch.cuda.mem_get_info(dev)
    geo = n * (3 * 40 + 1)
    ng = n * (640 + 1)
    staging = n * 4 * (2 * (49 + 52 + 10 + 2) + 3)  # double-buffered forward/gradient stage + plans
    render = a.width * a.height * 4 * 24 + (512 << 20)
    return "hbm" if 1.25 * (geo + ng + staging + render) < free else "host"


def link_probe(dev):
    """Measured pinned host<->device copy bandwidth (the host-offload tier's link roofline):
    1 GiB cudaMemcpyAsync each way, CUDA events, best of 3."""
    import torch

    nb = 1 << 30
    h = torch.empty(nb, dtype=torch.uint8).pin_memory()
    d = torch.empty(nb, dtype=torch.uint8, device=dev)
    out = {}
    for name, (dst, src) in (("h2d_gbs", (d, h)), ("d2h_gbs", (h, d))):
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, nb / (e0.elapsed_time(e1) / 1e3) / 1e9)
        out[name] = best
    del h, d
    torch.cuda.empty_cache()
    return out


def timed_engine(G, D, eng, a, dev, world, steps, warmup, kernel_timing=False):
    """W untimed warm-up iterations, then `steps` timed ones (barrier + device sync on both sides,
    CUDA events, max over ranks); the engine's stage and (optionally) per-kernel times."""
    import torch
    import torch.distributed as dist

    eng.run(warmup)
    eng.stage_ms()  # reset accumulators
    if kernel_timing:
        eng.kernel_timing(True)
        eng.kernel_times()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(torch.cuda.current_device())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    l0 = G.launch_count()
    losses, valid = eng.run(steps)
    launches = G.launch_count() - l0
    e1.record()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = D.max_over_ranks(e0.elapsed_time(e1), dev)
    stage = eng.stage_ms()
    kt = None
    if kernel_timing:
        kt = eng.kernel_times()
        eng.kernel_timing(False)
    return ms, losses, valid, launches, clocks, stage, kt


def run_ours(a, rank, world):
    import torch

    import paper_2509_15645_b200 as G
    from paper_2509_15645_b200 import dist as D

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # Weak scaling replicas: every rank owns an independent id-range shard of the scene (own seed)
    # and its optimizer state; no data-path collective.
    cfg = scene_config(a.n, a.width, a.height, a.cams, D.shard_seed(a.seed, rank))
    truth, cams = G.synth_scene_params(cfg)
    truth_dev = torch.from_numpy(truth).to(dev)
    gts = np.stack([G.render_view(truth_dev, c, 3).cpu().numpy() for c in cams])
    del truth_dev
    torch.cuda.empty_cache()
    start = training_start(truth)
    place = tier_placement(a, a.n, dev)
    eng = G.OffloadEngine(start, cams, gts, pipelined=True, nongeo_on_host=(place == "host"))

    # --- device-resident throughput (value), composite / sweep kernels timed live ---
    ms, losses, valid, launches, clocks, stage, kt = timed_engine(G, D, eng, a, dev, world, a.steps, a.warmup,
                                                                kernel_timing=True)
    ms_per_step = ms / a.steps
    value = world * a.steps / (ms / 1e3)

    # --- end to end through the public per-step API (host GT in, host loss out) ---
    # Headline: gss_engine_step_async — every step copies its pinned host GT in and its loss out to
    # pinned host memory; the host does not wait per step (the loss of step g lands while step g+1 is
    # enqueued). Also reported: the synchronous gss_engine_step (one host round trip per step).
    gts_pinned = [torch.from_numpy(g).pin_memory() for g in gts]
    ncam = len(cams)
    loss_pin = torch.zeros(max(a.steps, a.warmup), dtype=torch.float32).pin_memory()

    def e2e_loop(n, off, sync):
        for j in range(n):
            c = (off + j) % ncam
            if sync:
                eng.step(cams[c], gts_pinned[c].numpy())
            else:
                eng.step_async(cams[c], gts_pinned[c].view(-1), loss_pin[j:j + 1])
        eng.drain()

    res = {}
    for sync in (False, True):
        e2e_loop(a.warmup, 0, sync)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        e2e_loop(a.steps, a.warmup, sync)
        f1.record()
        torch.cuda.synchronize()
        res[sync] = D.max_over_ranks(f0.elapsed_time(f1), dev)
        if not sync:
            assert np.all(np.isfinite(loss_pin[:a.steps].numpy())) and float(loss_pin[a.steps - 1]) > 0
    e2e = {"value": world * a.steps / (res[False] / 1e3), "unit": "iters/s",
           "h2d_bytes_per_step": a.width * a.height * 3 * 4, "d2h_bytes_per_step": 4,
           "api": "gss_engine_step_async (OffloadEngine.step_async): pinned host GT -> loss in pinned host memory, "
                  "drained at the end of the timed region",
           "sync_step_value": world * a.steps / (res[True] / 1e3),
           "sync_step_api": "gss_engine_step: waits for each step's loss on the host"}
    eng.close()
    del eng
    torch.cuda.empty_cache()

    # --- the same workload with the non-geometric tier in pinned host memory (selective offload
    # over the host link: forwarding gather + lazy update cross PCIe) ---
    host = None
    if place != "host" and not a.no_host_offload and world == 1:
        h_steps, h_warm = min(a.steps, 6), min(a.warmup, 3)
        eng = G.OffloadEngine(start, cams, gts, pipelined=True, nongeo_on_host=True)
        hms, _, hvalid, _, hclocks, hstage, _ = timed_engine(G, D, eng, a, dev, world, h_steps, h_warm)
        eng.close()
        del eng
        torch.cuda.empty_cache()
        vis = float(np.mean(hvalid))
        touched = vis + (a.n - vis) / 16.0  # deferred update: grads + saturated counters (defer_max 15)
        link_bytes = vis * 3 * 196 + touched * 2 * 3 * 196  # counters stay in HBM
        host = {"value": h_steps / (hms / 1e3), "unit": "iters/s", "steps": h_steps, "warmup": h_warm,
                "ms_per_step": hms / h_steps, "stage_ms_per_step": {k: v / h_steps for k, v in hstage.items()},
                "clocks": hclocks, "link_bytes_per_step_est": link_bytes,
                "workload": "same scene, non-geometric tier (w/m/v) in pinned host memory, counters in HBM"}

    # --- isolated HBM-bound kernels on the trained state (culled/s; Adam GB/s) ---
    kern = [] if a.no_probe else kernel_probe(G, truth, cams, dev, a)
    link = link_probe(dev) if world == 1 else None
    if host is not None and link is not None:
        # link roofline of the host tier: the link bytes a step moves (forwarding gather reads the
        # visible rows' w/m/v + counters, the lazy pass reads and writes every touched row) over the
        # step time, against the measured copy peak of both directions (full duplex)
        ach = host["link_bytes_per_step_est"] / (host["ms_per_step"] / 1e3) / 1e9
        peak = link["h2d_gbs"] + link["d2h_gbs"]
        host["link_roofline"] = {"bound": "host link", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                                 "peak_source": "bench link probe: pinned cudaMemcpyAsync h2d + d2h (1 GiB, best of 3)"}

    vis = np.asarray(valid, np.float64)
    hbm, src = peaks()
    contribs_per_step = kt["contribs"] / max(a.steps, 1)
    out = {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference synth_scene generator, GT rendered on device)",
        "config": {"workload": (f"C4: synthetic {a.n / 1e6:g}M Gaussians, {a.width}x{a.height} views, selective offload "
                                f"(geometric tier in HBM, non-geometric tier in {'HBM (fits the budget)' if place == 'hbm' else 'pinned host memory'}), "
                                "pipelined, parameter forwarding, deferred Adam defer_max=15"),
                   "n_gaussians": a.n, "width": a.width, "height": a.height, "cams": a.cams, "nongeo_tier": place,
                   "parallelism": f"replicas x{world} (id-range shards, no data-path collective)" if world > 1
                   else "1 GPU", "l2": "inputs > L2 (30 GB optimizer state per rank at C4), no flush",
                   "mean_visible": float(vis.mean()), "used_ratio": float(vis.mean() / a.n),
                   "mean_contribs_per_px": contribs_per_step / (a.width * a.height)},
        "gpu_launches": int(launches),
        "stage_ms_per_step": {k: v / a.steps for k, v in stage.items()},
        "render_kernels": {"composite_ms_per_launch": kt["composite_ms"] / max(kt["composite_launches"], 1),
                           "sweep_ms_per_launch": kt["sweep_ms"] / max(kt["sweep_launches"], 1),
                           "contribs_per_step": contribs_per_step,
                           "composite_contribs_per_s": contribs_per_step / (kt["composite_ms"] / a.steps / 1e3),
                           "sweep_contribs_per_s": contribs_per_step / (kt["sweep_ms"] / a.steps / 1e3),
                           "composite_share_of_step": kt["composite_ms"] / ms, "sweep_share_of_step": kt["sweep_ms"] / ms,
                           # every timed render phase per step (CUDA events on stream D; the geometry
                           # phase includes the instance-count round trip to the host)
                           "phases_ms_per_step": {k: kt[f"{k}_ms"] / a.steps for k in
                                                  ("geometry", "colour", "composite", "sweep", "slot_sums", "chain")}},
        "kernels": kern,
        "e2e": e2e,
        "host_offload": host,
        "link": link,
        "clocks": clocks,
        "losses": [float(losses[0]), float(losses[-1])],
        "strips": "balanced by visible Gaussians per camera (imgpar.balanced_bounds)",
    }
    return out, (hbm, src), (cams, gts, start, truth)


def run_imgpar(a, rank, world):
    """N>1: every rank owns a contiguous id shard of one scene of N x a.n Gaussians
    (shard r = the reference generator at seed + r: the union is a scene N times denser), its
    optimizer state in HBM, and the column strip r of every view; each iteration renders the view
    image-parallel with two NCCL all-to-allv exchanges (splat records out, screen-space gradients
    back). Weak scaling: Gaussians per GPU fixed at a.n."""
    import torch
    import torch.distributed as dist

    import paper_2509_15645_b200 as G
    from paper_2509_15645_b200 import dist as D
    from paper_2509_15645_b200 import imgpar as IP

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % torch.cuda.device_count())
    dev = torch.device("cuda", torch.cuda.current_device())
    cfg = scene_config(a.n, a.width, a.height, a.cams, D.shard_seed(a.seed, rank))
    truth, cams = G.synth_scene_params(cfg)
    if world > 1:  # every rank renders the views of shard 0's generator
        obj = [[bytes(c) for c in cams]] if rank == 0 else [None]
        dist.broadcast_object_list(obj, src=0)
        cams = [G.camera_from_bytes(b) for b in obj[0]]
    ex = IP.TorchExchange() if world > 1 else IP.SelfExchange()
    # ground truth: the truth scene rendered image-parallel; this rank keeps its strip
    td = torch.from_numpy(truth).to(dev)
    geo_t, ng_t = td[:, :10].contiguous(), td[:, 10:].contiguous()
    gts = []
    for c in cams:
        vp = G.viewport_full(c.width, c.height)
        ids = G.frustum_cull(geo_t, geo_t.shape[0], c, vp)
        sc = G.RenderScene(ids=ids, geo=geo_t, nongeo=ng_t)
        _, _, strip, info = IP.render_step(ex, sc, c, vp, None)
        full = torch.zeros((c.height, c.width, 3), dtype=torch.float32, device=dev)
        b = info["bounds"]
        full[:, b[ex.rank]: b[ex.rank + 1]] = strip
        gts.append(full)
    del td, geo_t, ng_t
    torch.cuda.empty_cache()
    start = training_start(truth)
    # strips balanced by visible Gaussians over all shards; the loss stays on the device in the
    # timed loop (the e2e loop below reads it on the host every step)
    tr = IP.ShardTrainer(start, cams, gts, ex, pipelined=True, balance=True, device_loss=True)
    for _ in range(a.warmup):
        tr.step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(torch.cuda.current_device())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = G.launch_count()
    e0.record()
    losses, vis, sent = [], [], []
    for _ in range(a.steps):
        losses.append(tr.step())
        vis.append(tr.last_info["visible"])
        sent.append(tr.last_info["sent"])
    e1.record()
    torch.cuda.synchronize()
    launches = G.launch_count() - l0
    clocks = clk.stop()
    ms = D.max_over_ranks(e0.elapsed_time(e1), dev)
    # end to end: pinned host GT copied in every step, loss read back on the host
    # The next view's GT is prefetched on a copy stream into the other of two device buffers while
    # the current step runs (each step returns its loss on the host, so buffer j % 2 is free again
    # when step j + 1 is enqueued).
    pinned = [g.cpu().pin_memory() for g in gts]
    gbufs = [torch.empty_like(gts[0]), torch.empty_like(gts[0])]
    cstream = torch.cuda.Stream()
    ready = [torch.cuda.Event(), torch.cuda.Event()]

    def prefetch(j, view):
        with torch.cuda.stream(cstream):
            gbufs[j % 2].copy_(pinned[view % len(cams)], non_blocking=True)
            ready[j % 2].record(cstream)

    def e2e_loop(n, off):
        prefetch(0, off)
        for j in range(n):
            torch.cuda.current_stream().wait_event(ready[j % 2])
            if j + 1 < n:
                prefetch(j + 1, off + j + 1)
            float(tr.step(cams[(off + j) % len(cams)], gbufs[j % 2]))  # loss read on the host

    e2e_loop(a.warmup, 0)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    e2e_loop(a.steps, a.warmup)
    tr.drain()
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = D.max_over_ranks(f0.elapsed_time(f1), dev)
    hbm, src = peaks()
    vbar = float(np.mean(vis))
    out = {
        "metric": METRIC, "value": world * a.steps / (ms / 1e3), "unit": "iters/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference synth_scene generator per shard, GT rendered on device)",
        "config": {"workload": f"sharded: {world} x {a.n / 1e6:g}M Gaussians in one scene, "
                               f"{a.width}x{a.height} views rendered image-parallel ({world} column strips), "
                               "all state in HBM, deferred Adam defer_max=15",
                   "n_gaussians_per_gpu": a.n, "n_gaussians": a.n * world, "width": a.width, "height": a.height,
                   "cams": a.cams, "parallelism": f"id-range shards x{world} + image strips, NCCL all-to-allv"
                   if world > 1 else "1 GPU (split-phase path, no exchange)",
                   "l2": f"inputs > L2 ({a.n * 760 / 1e9:.1f} GB optimizer state per rank), no flush",
                   "mean_visible_per_gpu": vbar, "used_ratio": vbar / a.n,
                   "records_sent_per_gpu_per_step": float(np.mean(sent)),
                   "value_definition": "shard-iterations/s = N x (iterations/s of the N-shard job)"},
        "job_iters_per_s": a.steps / (ms / 1e3),
        "gpu_launches": int(launches),
        "e2e": {"value": world * a.steps / (e2e_ms / 1e3), "unit": "iters/s",
                "h2d_bytes_per_step": a.width * a.height * 3 * 4, "d2h_bytes_per_step": 8 * world + 8,
                "api": "imgpar.ShardTrainer.step: pinned host GT (next view prefetched on a copy stream) -> "
                       "loss on host every step"},
        "clocks": clocks,
        "losses": [float(losses[0]), float(losses[-1])],
    }
    return out, (hbm, src)


def kernel_probe(G, truth, cams, dev, a):
    """The HBM-bound kernels of the step launched alone on one stream, timed with CUDA events on
    that stream (average per launch): cull over the N x 10 geometric tier, the deferred Adam pass
    over the N x 49 non-geometric tier in steady state (>= 16 passes, 8.28% density, SURVEY.md
    §8d), the dense geo Adam pass over N x 10 and the forwarding gather (restore + pending)."""
    import ctypes as C

    import torch

    from paper_2509_15645_b200._abi import check, lib

    L = lib()
    n = a.n
    s = torch.cuda.current_stream()
    sp = s.cuda_stream
    reps = 20

    def timed(fn, reps=reps):
        for _ in range(3):
            fn(0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # Queue the launches behind a device-side spin so the host enqueue cost (ctypes + LUT
        # build per call) is off the timeline: the events then bracket back-to-back kernels.
        torch.cuda._sleep(20_000_000)
        e0.record(s)
        for r in range(reps):
            fn(r)
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    res = []
    # cull (render.hpp:253-260): B = 40 N + 4 V
    geo = torch.from_numpy(np.ascontiguousarray(truth[:, :10])).to(dev)
    ids = torch.empty(n, dtype=torch.int32, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    wsb = int(L.gss_cull_workspace_bytes(n))
    ws = torch.zeros(wsb, dtype=torch.uint8, device=dev)
    vp = G.viewport_full(a.width, a.height)
    cam0 = cams[0]

    def cull(_):
        check(L.gss_cull(geo.data_ptr(), n, 10, C.byref(cam0), C.byref(vp), 0.3, None, ids.data_ptr(),
                         cnt.data_ptr(), ws.data_ptr(), wsb, sp))

    ms = timed(cull)
    vis = int(cnt.item())
    b = 40 * n + 4 * vis
    res.append({"kernel": "cull_kernel", "op": "frustum_cull", "ms": ms, "bytes": b, "gbs": b / ms / 1e6,
                "culled_per_s": n / (ms / 1e3), "visible": vis})
    del geo, ws
    # deferred Adam, 49-wide non-geo tier (adam.hpp:211-238):
    # B = sum_touched 4*49*(6 + has_grad) + 2 N
    opt = G.OptimConfig()
    arena = G.Arena(n, 49, opt.nongeo_groups(), 15, device=dev, interleaved=True)  # the engine's layout
    arena.w.uniform_(-1, 1)
    dens = 0.0828
    gen = torch.Generator(device=dev)
    gen.manual_seed(7)
    nsched = 4
    sched = []
    for k in range(nsched):
        m = torch.rand(n, device=dev, generator=gen) < dens
        gi = torch.nonzero(m).flatten().to(torch.int32)
        # gradient rows in the engine's stage layout: 49 values in 52-float (16-byte aligned) rows
        sched.append((gi, torch.randn(gi.numel(), 52, device=dev, generator=gen)))
    # steady state: counters spread over [0, defer_max] (a long run's distribution; a fresh arena's
    # never-touched rows would all saturate in the same pass every 16th pass)
    arena.counter.copy_(torch.randint(0, 16, (n,), device=dev, generator=gen, dtype=torch.int32).to(torch.uint8))
    tcount = torch.zeros(reps + 8, dtype=torch.int64, device=dev)
    for k in range(20):
        G.deferred_update(arena, G.SparseGrads(sched[k % nsched][0], sched[k % nsched][1], 52), want_touched=False)
    st = arena.c_struct()
    gs = [G.SparseGrads(gi, gr, 52).c_struct() for gi, gr in sched]
    tot = {"t": 0, "g": 0}

    def deferred(r):
        g = gs[r % nsched]
        # touched rows of every timed pass land in their own slot (the byte model below)
        check(L.gss_deferred_update(C.byref(st), C.byref(g), None, tcount[r].data_ptr(), sp))

    ms = timed(deferred)
    arena._sync_step(st)
    touched_avg = float(tcount[:reps].double().mean().item())
    grads_avg = float(np.mean([gi.numel() for gi, _ in sched]))
    b = 4 * 49 * (6 * touched_avg + grads_avg) + 2 * n
    res.append({"kernel": "update_kernel + walk4_kernel (49-wide, deferred)", "op": "deferred_update", "ms": ms, "bytes": b,
                "gbs": b / ms / 1e6, "touched_rows": touched_avg, "grad_rows": grads_avg})
    # forwarding gather = restore_view with a pending pass (adam.hpp:252-289):
    # B = V (3*196 + 1) + V_pend * 196 + V * 196 (+ ids)
    gi, gr = sched[0]
    out = torch.empty(gi.numel(), 49, device=dev)
    pend = gs[1]

    def restore(_):
        check(L.gss_restore_view(C.byref(st), gi.data_ptr(), gi.numel(), None, C.byref(pend), out.data_ptr(), sp))

    ms = timed(restore)
    V = gi.numel()
    vp_ = sched[1][0].numel()
    b = V * (3 * 196 + 1 + 196 + 4) + vp_ * (196 + 4)
    res.append({"kernel": "restore_kernel (forwarding gather)", "op": "restore_view", "ms": ms, "bytes": b,
                "gbs": b / ms / 1e6, "rows": V})
    del arena, sched, gs, out
    torch.cuda.empty_cache()
    # geo Adam: dense pass over N x 10 with sparse grads (engine.hpp:380-386): B = 240 N + 40 V
    garena = G.Arena(n, 10, opt.geo_groups(), 0, device=dev)
    garena.w.uniform_(-1, 1)
    gi = torch.nonzero(torch.rand(n, device=dev, generator=gen) < dens).flatten().to(torch.int32)
    gg = torch.randn(gi.numel(), 10, device=dev, generator=gen)
    gst = garena.c_struct()
    ggs = G.SparseGrads(gi, gg, 10).c_struct()

    def geo_upd(_):
        check(L.gss_deferred_update(C.byref(gst), C.byref(ggs), None, None, sp))

    ms = timed(geo_upd)
    b = 240 * n + 44 * gi.numel()
    res.append({"kernel": "dense_update_kernel (10-wide, defer_max 0)", "op": "geo deferred_update (defer_max=0)", "ms": ms,
                "bytes": b, "gbs": b / ms / 1e6})
    del garena
    torch.cuda.empty_cache()
    return res


def load_traffic():
    """dram__bytes_read.sum + dram__bytes_write.sum per launch for the probed kernels, from the
    committed ncu --set full capture of this workload (profiles/); {} when absent."""
    f = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return {k: v["dram_bytes"] for k, v in json.loads(f.read_text()).items() if not k.startswith("_")}
    except Exception:
        return {}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# The reference rasterizer sample: REF_STRIPS full-width horizontal strips, evenly spaced, together
# REF_FRACTION of the image, plus one 16x16 window that measures the per-call cost independent of
# the window (project_all + the depth sort of all visible splats, render.hpp:402-411).
REF_STRIPS, REF_FRACTION = 4, 1.0 / 8.0


def _strips(w, h):
    sh = max(1, int(round(h * REF_FRACTION / REF_STRIPS)))
    out = []
    for k in range(REF_STRIPS):
        y0 = int((k + 0.5) * h / REF_STRIPS - sh / 2)
        out.append([0.0, float(w), float(y0), float(y0 + sh)])
    return out, REF_STRIPS * sh * w


def ref_stage_sample(O, start, gt_full, cam, a, workers, single_thread_render=False):
    """One bounded sample of a reference training iteration on this host (oracle/_ref/libgss_ref.so,
    the unmodified reference headers), timed stage by stage:
      cull            frustum_cull over all N geometric rows (render.hpp:253-260, single thread);
      forward_params  restore_view of the V visible rows with a pending gradient pass
                      (adam.hpp:252-289, single thread);
      render          rasterize_forward + compute_loss_l1 + rasterize_backward (render.hpp:384-640,
                      `workers` threads) on REF_STRIPS full-width strips covering REF_FRACTION of the
                      view (a full C4 view exceeds the renderer's int32 CSR, render.hpp:273), scaled to
                      the full view after subtracting the per-call cost t_fixed (project_all + depth
                      sort of all V splats, measured on a 16x16 window), which a view pays once;
      geo_update      deferred_update with defer_max 0 over N x 10 (engine.hpp:380-386);
      lazy_update     deferred_update, defer_max 15, N x 49, counters in steady state (adam.hpp:211-238).
    Gradient rows are synthetic N(0, 1e-3) and gt_full may be None (zeros): no stage's work depends
    on those values (the L1 gradient is nonzero at every covered pixel either way)."""
    import paper_2509_15645_b200 as G

    n = start.shape[0]
    W, H = a.width, a.height
    geo = np.ascontiguousarray(start[:, :10])
    t = {}
    c0 = time.perf_counter()
    ids = O.ref_cull(geo, cam, [0, W, 0, H])
    t["cull"] = time.perf_counter() - c0
    V = int(ids.size)
    opt = G.OptimConfig()
    grp = lambda gs: [(g.col0, g.dim, g.hp.lr) for g in gs]  # noqa: E731
    ng = O.RefArena(n, 49, grp(opt.nongeo_groups()), 15)
    ng.w[:] = start[:, 10:]
    rng = np.random.default_rng(7)
    ng.counter[:] = rng.integers(0, 16, n, dtype=np.uint8)  # steady-state counter spread
    ng.step = 32
    grads = (rng.standard_normal((V, 59), dtype=np.float32) * 1e-3)
    c0 = time.perf_counter()
    fwd = ng.restore(ids, pending=(ids, grads, 59, 10))
    t["forward_params"] = time.perf_counter() - c0
    gt = np.zeros((H, W, 3), np.float32) if gt_full is None else gt_full
    ngv = np.ascontiguousarray(fwd)

    def render(vp, workers_):
        c0 = time.perf_counter()
        r = O.render("ref", ids, geo, ngv, cam, vp, compact=True, gt=gt, normalizer=W * H * 3, workers=workers_)
        return time.perf_counter() - c0, r["contribs"]

    cx, cy = W // 2, H // 2
    t_fixed, _ = render([cx - 8.0, cx + 8.0, cy - 8.0, cy + 8.0], workers)
    strips, px = _strips(W, H)
    t_strips, contribs = 0.0, 0
    for vp in strips:
        dt, c = render(vp, workers)
        t_strips += dt
        contribs += c
    t["render"] = t_fixed + max(0.0, t_strips - len(strips) * t_fixed) * (W * H) / px
    sample = {"strips": len(strips), "pixels": px, "fraction": px / (W * H), "seconds": t_strips,
              "contribs": contribs, "t_fixed_s": t_fixed}
    ga = O.RefArena(n, 10, grp(opt.geo_groups()), 0)
    ga.w[:] = geo
    ga.step = 32
    c0 = time.perf_counter()
    ga.deferred(ids, grads, 59, 0)
    t["geo_update"] = time.perf_counter() - c0
    c0 = time.perf_counter()
    ng.deferred(ids, grads, 59, 10)
    t["lazy_update"] = time.perf_counter() - c0
    st1 = None
    if single_thread_render:  # one strip on one thread: the single-core rasterizer rate
        dt, c = render(strips[0], 1)
        st1 = {"seconds": dt, "contribs": c, "contribs_per_s": c / dt, "workers": 1}
    del ng, ga
    it = sum(t.values())
    return {"iteration_s": it, "stage_s": t, "visible": V, "render_sample": sample, "render_workers1_strip": st1}


def cpu_baseline(cams, gts, start, truth, a):
    """The reference's own CPU implementation (oracle/_ref/libgss_ref.so) timed on this host on a
    bounded sample of the same workload: ref_stage_sample on camera 0, all host threads."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles as O

    if O.ref() is None:
        return None
    cores = os.cpu_count() or 1
    cam = O.cam_from_struct(cams[0])
    t = time.perf_counter()
    r = ref_stage_sample(O, start, gts[0], cam, a, cores)
    dt = time.perf_counter() - t
    return {"value": 1.0 / r["iteration_s"], "unit": "iters/s", "cores": cores, "kind": "reference",
            "cpu": cpu_model(),
            "sample": f"camera 0 of the same {a.n / 1e6:g}M-Gaussian {a.width}x{a.height} workload: cull, forwarding "
                      "gather, geo and deferred Adam at full size (single-threaded in the reference), the "
                      "rasterizer fwd+loss+bwd (all cores) on 4 full-width strips = 1/8 of the view, scaled to the "
                      "full view (the reference's int32 CSR cannot hold a full C4 view)",
            "stage_s": r["stage_s"], "render_sample": r["render_sample"], "visible": r["visible"],
            "seconds": dt}


def run_reference(a, rank, world):
    """--impl reference: the reference CPU implementation on the same workload, rank 0 only. The
    scene comes from the reference's own generator (synth.hpp:100-154, via oracle ref_synth_nogt)
    and every stage runs in the reference library; no GPU and none of our code is used."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracles as O

    if rank != 0:
        return None
    if O.ref() is None:
        return {"impl": "reference", "unavailable": "oracle/_ref/libgss_ref.so not built (needs /root/reference)"}
    cfg = ref_scene_config(a)
    t0 = time.perf_counter()
    truth, cam_arr = O.ref_synth_nogt(cfg)
    t_synth = time.perf_counter() - t0
    start = training_start(truth)
    del truth
    cores = os.cpu_count() or 1
    w = min(a.warmup, 0)  # the CPU sample has no warm-up effects (no caches, no JIT)
    k = max(1, min(a.steps, a.ref_max_steps))
    its, runs = [], []
    t0 = time.perf_counter()
    for j in range(k):
        r = ref_stage_sample(O, start, None, cam_arr[j % len(cam_arr)], a, cores, single_thread_render=(j == 0))
        its.append(r["iteration_s"])
        runs.append(r)
    dt = time.perf_counter() - t0
    v = k / sum(its)
    return {"metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": world, "steps": k, "warmup": w,
            "ms_per_step": sum(its) / k * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (reference synth_scene generator)", "impl": "reference",
            "config": {"workload": f"C4: synthetic {a.n / 1e6:g}M Gaussians, {a.width}x{a.height} views, "
                                   "all state in host RAM (CPU reference), deferred Adam defer_max=15",
                       "n_gaussians": a.n, "width": a.width, "height": a.height, "cams": a.cams,
                       "requested_steps": a.steps, "requested_warmup": a.warmup,
                       "steps_cap": "each step is one bounded ~30-60 s sample of an iteration; capped at "
                                    f"--ref-max-steps={a.ref_max_steps} so the arm ends within minutes"},
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": cores, "kind": "reference", "cpu": cpu_model(),
                             "sample": f"{k} bounded iteration samples (cameras 0..{k - 1}): full-size cull, "
                                       "forwarding gather, geo + deferred Adam; rasterizer on 4 full-width strips "
                                       "(1/8 of the view) scaled to the full view (int32 CSR limit)"},
            "stages_s": [r["stage_s"] for r in runs], "render_sample": [r["render_sample"] for r in runs],
            "render_workers1_strip": runs[0]["render_workers1_strip"],
            "visible": [r["visible"] for r in runs], "synth_s": t_synth, "sample_wall_s": dt,
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def ref_scene_config(a):
    import paper_2509_15645_b200.gss as GS  # the config dataclass only (no library load)

    s = (1e5 / a.n) ** (1.0 / 3.0)
    return GS.SynthConfig(seed=a.seed, n=a.n, cams=a.cams, width=a.width, height=a.height, radius_min=1.5,
                          radius_max=3.0, scale_min=0.003 * s, scale_max=0.01 * s, fov_deg=30.0)


def spawn_ranks(a) -> int:
    """`--gpus N` (N > 1) without a torchrun environment: launch N ranks of this script on this
    node through torch.distributed.run (one process per GPU, rendezvous on 127.0.0.1), or fail
    loudly when fewer than N GPUs are visible — never silently run one rank."""
    import socket

    if a.impl == "ours":
        import torch

        have = torch.cuda.device_count()
        if have < a.gpus:
            sys.stderr.write(f"bench.py: --gpus {a.gpus} requested but only {have} CUDA device(s) visible\n")
            return 1
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        sys.exit(spawn_ranks(a))
    if world != a.gpus and "WORLD_SIZE" in os.environ:
        sys.stderr.write(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}\n")
        sys.exit(1)
    if world > 1:
        import torch.distributed as dist

        # GSS_BENCH_BACKEND=gloo: host-staged exchange (several ranks sharing one GPU, tests only)
        backend = os.environ.get("GSS_BENCH_BACKEND") or ("nccl" if a.impl == "ours" else "gloo")
        dist.init_process_group(backend)
    if a.impl == "reference":
        out = run_reference(a, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    mode = a.mode if a.mode != "auto" else ("engine" if world == 1 else "imgpar")
    if mode == "imgpar":
        out, _ = run_imgpar(a, rank, world)
        if rank == 0:
            print(json.dumps(out), flush=True)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()
        return
    out, (hbm, src), (cams, gts, start, truth) = run_ours(a, rank, world)
    if rank == 0:
        if out["kernels"]:
            out["culled_per_s"] = out["kernels"][0]["culled_per_s"]
        traffic = load_traffic()
        for kk in out["kernels"]:
            kk["frac"] = kk["gbs"] / hbm
            kk["traffic"] = traffic.get(kk["op"])
        out["roofline"] = render_roofline(out)
        if not a.no_cpu_baseline and world == 1:
            out["cpu_baseline"] = cpu_baseline(cams, gts, start, truth, a)
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


# Useful-work model of the dominant (SM-issue-bound) rasterizer kernel, from the committed
# profiles of the current kernels: the ncu issue-slot utilisation of the kernel and
# the fraction of the lane-pixel slots it issues that are useful contributions (a library built
# with GSS_RASTER_STATS=1, tools/raster_work.py).
RASTER_PROFILE = {
    "sweep": {"kernel": "backward_kernel", "issue_busy": 0.863, "useful_of_offered": 0.534,
              "dram_bytes_per_launch": 1.961671e9 + 1.389565e9,
              "source": "profiles/r02_ncu_sweep_c4_final.txt (Issue Slots Busy, dram__bytes of camera 0), "
                        "profiles/r02_raster_work_c4.json (bwd_useful_of_offered)"},
    "composite": {"kernel": "forward_kernel", "issue_busy": 0.856, "useful_of_offered": 0.655,
                  "dram_bytes_per_launch": 415.150848e6 + 265.354240e6,
                  "source": "profiles/r02_ncu_raster_c4_round2.txt (Issue Slots Busy, dram__bytes of camera 0), "
                            "profiles/r02_raster_work_c4.json (fwd_useful_of_offered)"},
}


def render_roofline(out):
    """Roofline of the step's dominant kernel: the rasterizer sweep or composite (whichever takes
    longer per step), both bound by SM instruction issue (no HBM or tensor-core roofline applies:
    DRAM < 3%, no contraction). achieved = useful contributions per launch / the launch's CUDA-event
    time measured live in the timed region; frac = issue-slot utilisation x useful fraction of the
    issued lane-pixel slots (the ceiling is every issue slot doing a useful contribution)."""
    rk = out["render_kernels"]
    which = "sweep" if rk["sweep_share_of_step"] >= rk["composite_share_of_step"] else "composite"
    prof = RASTER_PROFILE[which]
    ach = rk[f"{which}_contribs_per_s"]
    frac = prof["issue_busy"] * prof["useful_of_offered"]
    return {"bound": "issue", "kernel": prof["kernel"], "achieved": ach, "unit": "contribs/s",
            "peak": ach / frac, "frac": frac, "traffic": prof["dram_bytes_per_launch"],
            "traffic_note": "ncu dram__bytes_read + write of one launch (camera 0): < 5% of HBM bandwidth over "
                            "the launch, so neither kernel is memory-bound",
            "share_of_step": rk[f"{which}_share_of_step"],
            "bytes_or_units_per_launch": rk["contribs_per_step"],
            "frac_source": prof["source"],
            "note": "units = (pixel, splat) contributions composited per view (SURVEY.md §8a rows a8/a10); "
                    "HBM-bound kernels (cull, deferred Adam, gather, geo Adam) are in `kernels` with their "
                    "fraction of the measured HBM peak"}


if __name__ == "__main__":
    main()
