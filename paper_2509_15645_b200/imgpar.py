"""Image-parallel rendering and sharded training over N GPUs.

Partition: Gaussians and all their optimizer state by contiguous id range (dist.id_range), so cull,
forwarding gather and both Adam passes are shard-local. A view is rendered image-parallel:

  A  owner:  project its visible Gaussians into 64-byte splat records (gss_project) and route each
             record to every column strip its pixel box touches (gss_route_strips), ascending slots;
  X1 all-to-allv of records (NCCL over NVLink; ranks concatenate what they receive in rank order,
             which is ascending global id because shards are ascending id ranges);
  B  strip:  composite the received records on its strip (gss_rasterize_records_forward): the
             per-pixel contribution lists are the unsplit ones, so strip pixels are bit-identical;
             the loss is the fp64 sum of the strips' fp64 |d| sums, cast once (render.hpp:510);
  C  strip:  backward -> one 9-float screen-space gradient sum per received record (the SlotAcc
             cut of render.hpp:538);
  X2 all-to-allv back to the owners (the reverse splits of X1);
  D  owner:  sum the strips' partials per slot in strip order (gss_scatter_add_rows, fixed order:
             deterministic) and run the per-Gaussian chain locally (gss_chain_backward).

The reference's batch-1 semantics are kept (no view batching). Confined Gaussians' gradients are
the unsplit ones up to the tile-partial association; straddlers reassociate like the reference's
own split aggregation (splitter.hpp:85-123, pinned at <= 1e-5 by test_split.cpp:144-211).

`simulate_render` runs the same phases for R virtual shards in one process (the exchange is a
concatenation): the single-GPU parity harness of the multi-GPU path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import gss as G
from ._abi import GssViewport


def strip_bounds(px0: int, pw: int, nstrips: int, align: int = 16) -> List[int]:
    """Column boundaries of `nstrips` strips over pixels [px0, px0 + pw): whole 16-pixel tiles,
    sizes differing by at most one tile (the last strip absorbs the ragged edge)."""
    if nstrips < 1:
        raise ValueError("strip_bounds: nstrips must be >= 1")
    tiles = -(-pw // align)
    base, extra = divmod(tiles, nstrips)
    b = [px0]
    for k in range(nstrips):
        b.append(min(px0 + pw, b[-1] + (base + (1 if k < extra else 0)) * align))
    b[-1] = px0 + pw
    return b


def strip_viewport(vp: GssViewport, bounds: Sequence[int], k: int) -> GssViewport:
    """The viewport whose pixel window (render.hpp:297-304) is columns [bounds[k], bounds[k+1])."""
    return GssViewport(float(bounds[k]), float(bounds[k + 1]), vp.y0, vp.y1)


def window_of(vp: GssViewport) -> Tuple[int, int, int, int]:
    import math
    px0 = max(int(math.ceil(float(np.float32(vp.x0)) - 0.5)), 0)
    py0 = max(int(math.ceil(float(np.float32(vp.y0)) - 0.5)), 0)
    pw = max(0, int(math.ceil(float(np.float32(vp.x1)) - 0.5)) - px0)
    ph = max(0, int(math.ceil(float(np.float32(vp.y1)) - 0.5)) - py0)
    return px0, py0, pw, ph


def loss_from_sums_dev(parts: torch.Tensor, normalizer: int) -> torch.Tensor:
    """loss_from_sums on the device (no host round trip): the fp64 strip sums added in strip order,
    cast once, times (float)(1 / normalizer) — the same arithmetic, a float32 scalar tensor."""
    tot = parts[0]
    for k in range(1, int(parts.shape[0])):
        tot = tot + parts[k]
    inv = torch.tensor(float(np.float32(1.0) / np.float32(float(normalizer))), dtype=torch.float32, device=parts.device)
    return tot.to(torch.float32) * inv


def loss_from_sums(sums_f64: Sequence[float], normalizer: int) -> float:
    """(float)(sum of the strips' fp64 sums, in strip order) * (1 / (float)normalizer), the device
    loss_final arithmetic (render.hpp:510)."""
    tot = 0.0
    for s in sums_f64:
        tot += float(s)
    inv = np.float32(1.0) / np.float32(float(normalizer))
    return float(np.float32(tot) * inv)


# ------------------------------------------------------------------------------------------------
# Phases (one shard / one strip each; device tensors)

@dataclass
class OwnerState:
    scene: G.RenderScene
    recs: torch.Tensor  # [V, 64] uint8
    slots: torch.Tensor  # [R, V] int32 (row k: first counts[k] entries)
    counts: List[int]


def owner_project(scene: G.RenderScene, cam, vp: GssViewport, bounds: Sequence[int]):
    """Phase A: records of this shard's visible slots and the send buffer (strip-major, ascending
    slots within a strip). Returns (state, send [sum counts, 64] uint8, send counts)."""
    recs = G.project(scene, cam, vp)
    slots, counts = G.route_strips(recs, bounds)
    sel = torch.cat([slots[k, : counts[k]] for k in range(len(counts))]) if recs.shape[0] else \
        torch.zeros(0, dtype=torch.int32, device=recs.device)
    send = G.gather_records(recs, sel)
    return OwnerState(scene, recs, slots, counts), send, counts


def strip_forward(recv: torch.Tensor, cam, vp_strip: GssViewport, background, gt: Optional[torch.Tensor],
                  normalizer: int) -> G.RecordsResult:
    """Phase B: composite the received records on the strip (loss/d_img fused when gt is given)."""
    return G.rasterize_records_forward(recv, cam, vp_strip, background=background, gt=gt, normalizer=normalizer)


def strip_backward(fw: G.RecordsResult, d_img: torch.Tensor) -> torch.Tensor:
    """Phase C: per-received-record 9-float screen-space gradient sums."""
    return G.rasterize_records_backward(fw, d_img)


def owner_combine(st: OwnerState, back: torch.Tensor) -> torch.Tensor:
    """Phase D (first half): per-slot sums of the strips' returned partials in strip order."""
    V = int(st.recs.shape[0])
    sums = torch.zeros((max(V, 1), 9), dtype=torch.float32, device=st.recs.device)[:V]
    off = 0
    for k, c in enumerate(st.counts):
        if c:
            G.scatter_add_rows(back[off: off + c], st.slots[k, :c], sums)
        off += c
    return sums


def owner_chain(st: OwnerState, cam, sums: torch.Tensor) -> G.GradBuffer:
    """Phase D (second half): the per-Gaussian chain on the owner."""
    return G.chain_backward(st.scene, cam, st.recs, sums)


# ------------------------------------------------------------------------------------------------
# Exchange over torch.distributed

class TorchExchange:
    """all-to-allv / all-gather over a torch.distributed group. With NCCL the device tensors go
    over NVLink directly; with any other backend (gloo: CPU tests, or several processes sharing
    one GPU) they are staged through host memory."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device_native = dist.get_backend(group) == "nccl"

    def _dev(self, t: torch.Tensor) -> torch.Tensor:
        return t if self.device_native else t.cpu()

    def alltoallv(self, send: torch.Tensor, send_counts: Sequence[int],
                  recv_counts: Optional[Sequence[int]] = None) -> Tuple[torch.Tensor, List[int]]:
        """Rows send[sum(send_counts[:j]) : +send_counts[j]] go to rank j; returns the rows
        received, concatenated in rank order, and their counts."""
        d = self.dist
        if recv_counts is None:
            dev = send.device if self.device_native else "cpu"
            sc = torch.tensor([int(c) for c in send_counts], dtype=torch.int64, device=dev)
            rc = torch.empty_like(sc)
            d.all_to_all_single(rc, sc, group=self.group)
            recv_counts = rc.cpu().tolist()
        recv_counts = [int(c) for c in recv_counts]
        out = torch.empty((sum(recv_counts),) + tuple(send.shape[1:]), dtype=send.dtype,
                          device=send.device if self.device_native else "cpu")
        d.all_to_all_single(out, self._dev(send.contiguous()), output_split_sizes=recv_counts,
                            input_split_sizes=[int(c) for c in send_counts], group=self.group)
        return out.to(send.device), recv_counts

    def allgather_f64(self, x: torch.Tensor) -> List[float]:
        return [float(v) for v in self.allgather_f64_dev(x).cpu().tolist()]

    def allgather_f64_dev(self, x: torch.Tensor) -> torch.Tensor:
        """[world] fp64 tensor on x's device (rank order); no host round trip with NCCL."""
        t = x.reshape(1).to(torch.float64)
        t = t if self.device_native else t.cpu()
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        return torch.cat(parts).to(x.device)


def render_step(ex: TorchExchange, scene: G.RenderScene, cam, vp: GssViewport, gt: Optional[torch.Tensor],
                background=(0.0, 0.0, 0.0), normalizer: int = 0, bounds: Optional[Sequence[int]] = None,
                device_loss: bool = False):
    """One view, image-parallel over the exchange group: returns (loss, GradBuffer of this shard,
    strip image, info). Rank k owns strip k of `vp` (column bounds: `bounds`, e.g. the balanced
    ones of balanced_bounds, else equal whole-tile strips). device_loss: the loss stays a device
    float32 scalar (no host round trip)."""
    px0, py0, pw, ph = window_of(vp)
    bounds = list(bounds) if bounds is not None else strip_bounds(px0, pw, ex.world)
    if len(bounds) != ex.world + 1 or bounds[0] != px0 or bounds[-1] != px0 + pw:
        raise ValueError("render_step: bounds must be world + 1 column cuts spanning the window")
    norm = normalizer if normalizer > 0 else pw * ph * 3
    st, send, scounts = owner_project(scene, cam, vp, bounds)
    recv, rcounts = ex.alltoallv(send, scounts)
    fw = strip_forward(recv, cam, strip_viewport(vp, bounds, ex.rank), background, gt, norm)
    loss = None
    if gt is not None:
        if device_loss:
            loss = loss_from_sums_dev(ex.allgather_f64_dev(fw.loss_sum), norm)
        else:
            loss = loss_from_sums(ex.allgather_f64(fw.loss_sum), norm)
    part = strip_backward(fw, fw.d_img) if gt is not None else None
    gb = None
    if part is not None:
        back, _ = ex.alltoallv(part, rcounts, recv_counts=scounts)
        gb = owner_chain(st, cam, owner_combine(st, back))
    info = dict(sent=sum(scounts), received=sum(rcounts), instances=fw.instances, bounds=bounds)
    return loss, gb, fw.image, info


def simulate_render(scenes: Sequence[G.RenderScene], cam, vp: GssViewport, gt: Optional[torch.Tensor],
                    background=(0.0, 0.0, 0.0), normalizer: int = 0):
    """R = len(scenes) virtual shards in one process, same phases, exchange = concatenation.
    Returns (loss, [GradBuffer per shard], full image assembled from the strips)."""
    R = len(scenes)
    px0, py0, pw, ph = window_of(vp)
    bounds = strip_bounds(px0, pw, R)
    norm = normalizer if normalizer > 0 else pw * ph * 3
    owners = [owner_project(sc, cam, vp, bounds) for sc in scenes]
    offs = [np.concatenate([[0], np.cumsum(o[2])]).astype(np.int64) for o in owners]
    fws, recv_counts = [], []
    for k in range(R):
        parts = [o[1][offs[r][k]: offs[r][k + 1]] for r, o in enumerate(owners)]
        recv_counts.append([int(p.shape[0]) for p in parts])
        recv = torch.cat(parts) if parts else owners[0][1][:0]
        fws.append(strip_forward(recv, cam, strip_viewport(vp, bounds, k), background, gt, norm))
    image = torch.cat([f.image for f in fws], dim=1)
    loss = loss_from_sums([float(f.loss_sum.item()) for f in fws], norm) if gt is not None else None
    grads = None
    if gt is not None:
        parts_back = [strip_backward(f, f.d_img) for f in fws]
        grads = []
        for r, (st, _, scounts) in enumerate(owners):
            segs = []
            for k in range(R):
                o = int(sum(recv_counts[k][:r]))
                segs.append(parts_back[k][o: o + recv_counts[k][r]])
            back = torch.cat(segs)
            grads.append(owner_chain(st, cam, owner_combine(st, back)))
    return loss, grads, image


class SelfExchange:
    """The exchange of a single rank (world 1): every send segment comes straight back."""

    rank, world = 0, 1

    def alltoallv(self, send, send_counts, recv_counts=None):
        return send, [int(c) for c in send_counts]

    def allgather_f64(self, x):
        return [float(x.reshape(-1)[0].item())]

    def allgather_f64_dev(self, x):
        return x.reshape(1).to(torch.float64)


def balanced_bounds(ex, geo: torch.Tensor, n: int, cam, vp: GssViewport, align: int = 16) -> List[int]:
    """Column strips balanced by visible Gaussians over all shards (evalsplit.balanced_strip_bounds,
    the reference's split search generalised to N strips, splitter.hpp:31-81): each evaluation is
    an exact device cull of this shard for viewport [px0, c), summed over the exchange group."""
    from . import evalsplit as ES

    px0, py0, pw, ph = window_of(vp)

    def count_upto(c):
        sub = GssViewport(vp.x0, float(c), vp.y0, vp.y1)
        local = torch.tensor([float(G.frustum_cull(geo, n, cam, sub).numel())], dtype=torch.float64,
                             device=geo.device)
        return int(round(sum(ex.allgather_f64(local))))

    return ES.balanced_strip_bounds(count_upto, px0, pw, ex.world, align)


class ShardTrainer:
    """One rank of sharded training: this rank's contiguous id shard of the scene
    with its geometric (dense, geo_defer_max 0) and non-geometric (deferred, defer_max) Adam arenas
    in HBM, and the reference engine's per-iteration DAG in run_serial order (engine.hpp:434-445):

        cull(g) -> forward_params(g) [restore_view with pending grads(g-1)] -> lazy(g-1)
        -> render(g) [image-parallel over the exchange group] -> geo_update(g)

    Every stage is shard-local except the render's two all-to-allv exchanges. With one rank and
    SelfExchange the trajectory equals OffloadEngine(pipelined=False) on the same shard. pipelined=True
    runs forward_params(g) and lazy(g-1) on a second CUDA stream (the engine's stream H,
    engine.hpp:464-522) so the lazy update overlaps render(g); the results are bitwise the same."""

    def __init__(self, init_rows: np.ndarray, cams, gts, ex=None, optim: Optional[G.OptimConfig] = None, *,
                 sh_degree: int = 3, sh_warmup_step: int = 0, background=(0.0, 0.0, 0.0), device=None,
                 pipelined: bool = False, balance: bool = False, device_loss: bool = False):
        """balance: per-camera strips balanced by visible Gaussians (balanced_bounds, computed on
        the camera's first use) instead of equal column strips. device_loss: step() returns the
        loss as a device float32 scalar (no per-step host round trip for it)."""
        self.ex = ex or SelfExchange()
        self.balance = bool(balance)
        self.device_loss = bool(device_loss)
        self.bounds = {}
        self.pipelined = bool(pipelined)
        self.sH = torch.cuda.Stream() if self.pipelined else None
        self.opt = optim or G.OptimConfig()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        rows = torch.from_numpy(np.ascontiguousarray(init_rows, np.float32)).to(dev)
        self.n = int(rows.shape[0])
        self.geo = G.Arena(self.n, G.K_GEO_DIM, self.opt.geo_groups(), self.opt.geo_defer_max, device=dev)
        self.ng = G.Arena(self.n, G.K_NONGEO_DIM, self.opt.nongeo_groups(), self.opt.defer_max, device=dev,
                          interleaved=True)
        self.geo.w.copy_(rows[:, : G.K_GEO_DIM])
        self.ng.w.copy_(rows[:, G.K_GEO_DIM:])
        del rows
        self.cams = list(cams)
        self.gts = gts  # per camera: device tensor (H x W x 3; only this rank's strip is read) or None
        self.sh_degree, self.sh_warmup_step = int(sh_degree), int(sh_warmup_step)
        self.background = tuple(float(b) for b in background)
        self.g = 0
        self.pending: Optional[G.SparseGrads] = None
        self.last_info = {}
        # densification statistics of this shard (engine.hpp:404-408: accum_norm += |dL/dmean2d|,
        # accum_cnt += 1 per visible Gaussian per iteration), as the engine's handoff stage keeps them
        self.accum_norm = torch.zeros(max(self.n, 1), dtype=torch.float64, device=dev)[: self.n]
        self.accum_cnt = torch.zeros(max(self.n, 1), dtype=torch.int32, device=dev)[: self.n]

    def step(self, cam=None, gt: Optional[torch.Tensor] = None) -> float:
        g = self.g
        cam = cam if cam is not None else self.cams[g % len(self.cams)]
        gt = gt if gt is not None else self.gts[g % len(self.cams)]
        vp = G.viewport_full(cam.width, cam.height)
        ids = G.frustum_cull(self.geo.w, self.n, cam, vp)                      # cull(g)
        if self.pipelined:
            main, sH = torch.cuda.current_stream(), self.sH
            sH.wait_stream(main)  # ids(g) and the pending grads(g-1) are ready
            ids.record_stream(sH)
            with torch.cuda.stream(sH):
                fwd = G.restore_view(self.ng, ids, self.pending, stream=sH)    # forward_params(g)
                ev_fp = torch.cuda.Event()
                ev_fp.record(sH)
                if self.pending is not None:                                   # lazy(g-1), overlaps render(g)
                    self.pending.ids.record_stream(sH)
                    self.pending.rows.record_stream(sH)
                    G.deferred_update(self.ng, self.pending, want_touched=False, check_invariants=False, stream=sH)
            fwd.record_stream(main)
            main.wait_event(ev_fp)
        else:
            fwd = G.restore_view(self.ng, ids, self.pending)                   # forward_params(g)
            if self.pending is not None:                                       # lazy(g-1)
                G.deferred_update(self.ng, self.pending, want_touched=False, check_invariants=False)
        deg = min(self.sh_degree, g // self.sh_warmup_step) if self.sh_warmup_step > 0 else self.sh_degree
        sc = G.RenderScene(ids=ids, geo=self.geo.w, nongeo=fwd, nongeo_compact=True, sh_degree=deg,
                           background=self.background)
        bounds = None
        if self.balance:
            ci = g % len(self.cams) if cam is self.cams[g % len(self.cams)] else None
            key = ci if ci is not None else id(cam)
            if key not in self.bounds:
                self.bounds[key] = balanced_bounds(self.ex, self.geo.w, self.n, cam, vp)
            bounds = self.bounds[key]
        loss, gb, _, info = render_step(self.ex, sc, cam, vp, gt, self.background, bounds=bounds,
                                        device_loss=self.device_loss)  # render(g)
        G.deferred_update(self.geo, G.SparseGrads(ids, gb.rows, G.K_PARAM_DIM, 0), want_touched=False,
                          check_invariants=False)                              # geo_update(g)
        self.pending = G.SparseGrads(ids, gb.rows, G.K_PARAM_DIM, G.K_GEO_DIM)  # handoff(g)
        if ids.numel():  # densification statistics (engine.hpp:404-408), fp64, ids unique
            m = gb.mean2d.reshape(-1, 2).double()
            idl = ids.long()
            self.accum_norm.index_add_(0, idl, torch.sqrt(m[:, 0] * m[:, 0] + m[:, 1] * m[:, 1]))
            self.accum_cnt.index_add_(0, idl, torch.ones_like(ids))
        self.last_info = dict(info, visible=int(ids.numel()))
        self.g += 1
        return loss

    def drain(self) -> None:
        if self.pipelined:
            torch.cuda.current_stream().wait_stream(self.sH)
        if self.pending is not None:
            G.deferred_update(self.ng, self.pending, want_touched=False, check_invariants=False)
            self.pending = None
        if self.pipelined:  # the non-geometric arena was last written on stream H
            torch.cuda.current_stream().wait_stream(self.sH)

    def state(self):
        return dict(geo_w=self.geo.w, ng_w=self.ng.w, ng_m=self.ng.m, ng_v=self.ng.v, ng_counter=self.ng.counter)
