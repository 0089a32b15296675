"""Reference-shaped Python API over libgss_b200 (device tensors in, device tensors out).

Names, argument meaning and errors mirror /root/reference/proj/include/gss/*.hpp so code written
against the reference path reads the same:

    frustum_cull        render.hpp:253-260
    rasterize_forward   render.hpp:384-464   (RenderResult keeps the device aux for backward)
    compute_loss_l1     render.hpp:497-511
    rasterize_backward  render.hpp:526-640   (GradBuffer: ids, rows V x 59, mean2d V x 2)
    build_group_luts    adam.hpp:67-97
    Arena / adam_step_dense / deferred_update / restore_view / flush_deferred   adam.hpp:119-313
    OffloadEngine       engine.hpp:55-522

Torch is used only for device memory and the current stream; every computation is a call into
the sm_100a kernels of libgss_b200.so.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from ._abi import (GssArena, GssCamera, GssDensifyConfig, GssEngineConfig, GssGroup, GssRenderScene, GssSparseGrads, GssViewport,
                   ConfigError, InvariantViolation, check, lib)

K_GEO_DIM, K_NONGEO_DIM, K_PARAM_DIM = 10, 49, 59
K_LOW_PASS = 0.3


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dev(device=None) -> torch.device:
    return torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())


# ---------------------------------------------------------------------------------------------
# Camera / Viewport (scene.hpp:77-96, render.hpp:45-49)

def camera(rot, trans, fx, fy, cx, cy, width, height, near_plane, far_plane) -> GssCamera:
    c = GssCamera()
    r = np.asarray(rot, dtype=np.float32).reshape(9)
    t = np.asarray(trans, dtype=np.float32).reshape(3)
    for i in range(9):
        c.rot[i] = float(r[i])
    for i in range(3):
        c.trans[i] = float(t[i])
    c.fx, c.fy, c.cx, c.cy = float(fx), float(fy), float(cx), float(cy)
    c.width, c.height = int(width), int(height)
    c.near_plane, c.far_plane = float(near_plane), float(far_plane)
    return c


def camera_from_bytes(b: bytes) -> GssCamera:
    return GssCamera.from_buffer_copy(b)


def look_at_camera(eye, target, fx, fy, w, h, near_p, far_p) -> GssCamera:
    e = (C.c_float * 3)(*map(float, eye))
    t = (C.c_float * 3)(*map(float, target))
    out = GssCamera()
    check(lib().gss_look_at_camera(e, t, float(fx), float(fy), int(w), int(h), float(near_p), float(far_p),
                                   C.byref(out)))
    return out


def viewport_full(w: int, h: int) -> GssViewport:
    return GssViewport(0.0, float(w), 0.0, float(h))


# ---------------------------------------------------------------------------------------------
# Culling

def cull_workspace_bytes(n: int) -> int:
    return int(lib().gss_cull_workspace_bytes(int(n)))


def frustum_cull(geo: torch.Tensor, count: int, cam: GssCamera, vp: GssViewport, low_pass: float = K_LOW_PASS,
                 *, stride: Optional[int] = None, want_mask: bool = False, stream=None, sync: bool = True):
    """frustum_cull (render.hpp:253-260): ascending kept ids (int32 device tensor).

    With sync=False returns (ids_capacity_tensor, count_dev, mask) without reading the count."""
    assert geo.is_cuda and geo.dtype == torch.float32
    stride = stride if stride is not None else (geo.shape[1] if geo.dim() == 2 else K_GEO_DIM)
    dev = geo.device
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    if st != torch.cuda.current_stream(dev):
        st.wait_stream(torch.cuda.current_stream(dev))  # geo written on the caller's stream
    # Outputs and the zero-filled workspace are allocated (and zeroed) on the launch stream, so the
    # caching allocator orders their reuse after the cull.
    with torch.cuda.stream(st):
        ids = torch.empty(max(count, 1), dtype=torch.int32, device=dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=dev)
        ws = torch.zeros(cull_workspace_bytes(count), dtype=torch.uint8, device=dev)
        mask = torch.empty(max((count + 31) // 32, 1), dtype=torch.int32, device=dev) if want_mask else None
        check(lib().gss_cull(_ptr(geo), int(count), int(stride), C.byref(cam), C.byref(vp), float(low_pass),
                             _ptr(mask), _ptr(ids), _ptr(cnt), _ptr(ws), ws.numel(), st.cuda_stream))
        lib().gss_cull_workspace_release(_ptr(ws))
    geo.record_stream(st)
    if not sync:
        return ids, cnt, mask
    st.synchronize()
    v = int(cnt.item())
    ids = ids[:v]
    return (ids, mask) if want_mask else ids


# ---------------------------------------------------------------------------------------------
# Optimizer

@dataclass
class Hyperparams:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8

    def validate(self) -> None:  # adam.hpp:20-25
        if not self.lr > 0:
            raise ConfigError(2, "hyperparams: lr must be > 0")
        if not (0 <= self.beta1 < 1):
            raise ConfigError(2, "hyperparams: require 0 <= beta1 < 1")
        if not (0 <= self.beta2 < 1):
            raise ConfigError(2, "hyperparams: require 0 <= beta2 < 1")
        if not self.eps > 0:
            raise ConfigError(2, "hyperparams: eps must be > 0")


@dataclass
class GroupSpec:
    name: str
    col0: int
    dim: int
    hp: Hyperparams = field(default_factory=Hyperparams)


@dataclass
class GroupLuts:
    param: np.ndarray
    mom: np.ndarray
    var: np.ndarray
    pow_b1: np.ndarray
    pow_b2: np.ndarray
    one_minus_b1: float
    one_minus_b2: float
    bias_correction: float
    step_size: float
    eps: float


def build_group_luts(hp: Hyperparams, t: int, max_delay: int) -> GroupLuts:
    arrs = [np.zeros(max_delay + 1, np.float32) for _ in range(5)]
    sc = np.zeros(5, np.float32)
    p = [a.ctypes.data for a in arrs]
    check(lib().gss_build_group_luts(hp.lr, hp.beta1, hp.beta2, hp.eps, int(t), int(max_delay), *p,
                                     sc.ctypes.data))
    return GroupLuts(*arrs, *map(float, sc))


class Arena:
    """Arena<float> (adam.hpp:119-159) resident in device memory: w, m, v [n, dim] + uint8 counter."""

    def __init__(self, n: int, dim: int, groups: Sequence[GroupSpec], defer_max: int, device=None, *,
                 interleaved: bool = False, host: bool = False):
        """host=True: the row-interleaved w/m/v buffer in pinned host memory (the offload tier,
        store.hpp:149-192; counters stay on the device) — passes over it are staged through HBM."""
        if host and not interleaved:
            raise ConfigError(2, "arena: a host-resident arena uses the row-interleaved layout")
        if defer_max < 0 or defer_max > 254:
            raise ConfigError(2, "arena: defer max must be in [0, 254]")
        covered = 0
        for g in groups:
            g.hp.validate()
            covered += g.dim
        if covered != dim:
            raise ConfigError(2, "arena: group dims must cover the row")
        dev = _dev(device)
        self.count, self.dim, self.groups, self.defer_max = int(n), int(dim), list(groups), int(defer_max)
        if interleaved:
            # one row-interleaved buffer: [w | m | v | pad] per row, each segment padded to whole
            # float4s (16-byte aligned), the row to whole 128-byte lines (the engine's layout)
            seg = -(-dim // 4) * 4
            self.row_stride = -(-3 * seg // 32) * 32
            if host:
                self._buf = torch.zeros((n, self.row_stride), dtype=torch.float32).pin_memory()
            else:
                self._buf = torch.zeros((n, self.row_stride), dtype=torch.float32, device=dev)
            self.w, self.m, self.v = (self._buf[:, i * seg:i * seg + dim] for i in range(3))
        else:
            self.row_stride = dim
            self.w = torch.zeros((n, dim), dtype=torch.float32, device=dev)
            self.m = torch.zeros((n, dim), dtype=torch.float32, device=dev)
            self.v = torch.zeros((n, dim), dtype=torch.float32, device=dev)
        self.counter = torch.zeros(max(n, 1), dtype=torch.uint8, device=dev)[:n]
        self.step = 0
        self.host = bool(host)

    def __del__(self):
        # the library's scratch + sticky error flag for this arena (keyed by the counter buffer)
        c = getattr(self, "counter", None)
        if c is not None:
            try:
                a = GssArena()
                a.counter = _ptr(c)
                lib().gss_arena_release(C.byref(a))
            except Exception:
                pass

    def c_struct(self) -> GssArena:
        a = GssArena()
        a.w, a.m, a.v, a.counter = _ptr(self.w), _ptr(self.m), _ptr(self.v), _ptr(self.counter)
        a.n, a.dim, a.defer_max, a.step = self.count, self.dim, self.defer_max, self.step
        a.row_stride = self.row_stride
        a.ngroups = len(self.groups)
        for i, g in enumerate(self.groups):
            a.groups[i] = GssGroup(g.col0, g.dim, g.hp.lr, g.hp.beta1, g.hp.beta2, g.hp.eps)
        return a

    def _sync_step(self, a: GssArena) -> None:
        self.step = int(a.step)

    def access(self) -> dict:
        """AccessReport (adam.hpp:36-50) tallied on the device since the arena's first use."""
        out = np.zeros(6, np.uint64)
        a = self.c_struct()
        check(lib().gss_arena_access(C.byref(a), out.ctypes.data))
        return dict(zip(("update_passes", "touched_rows", "param_bytes", "counter_bytes", "restore_rows",
                         "restore_read_bytes"), (int(x) for x in out)))

    def check_counters(self, stream=None) -> None:
        """check_counters (adam.hpp:154-158) + the sortedness flag of the last deferred pass."""
        a = self.c_struct()
        check(lib().gss_arena_check(C.byref(a), _stream(stream)))


@dataclass
class SparseGrads:
    """SparseGrads<float> (adam.hpp:163-169): sorted ids; row(k) = rows[k*stride + col0 ...]."""

    ids: torch.Tensor
    rows: Optional[torch.Tensor]
    stride: int
    col0: int = 0
    count_dev: Optional[torch.Tensor] = None

    def c_struct(self) -> GssSparseGrads:
        g = GssSparseGrads()
        g.ids = _ptr(self.ids) if self.ids is not None and self.ids.numel() else None
        g.count = int(self.ids.numel()) if self.ids is not None else 0
        g.count_dev = _ptr(self.count_dev)
        g.rows = _ptr(self.rows) if self.rows is not None and self.rows.numel() else None
        g.stride, g.col0 = int(self.stride), int(self.col0)
        return g


def adam_step_dense(a: Arena, grads: Optional[torch.Tensor], stream=None) -> None:
    s = a.c_struct()
    check(lib().gss_adam_step_dense(C.byref(s), _ptr(grads), _stream(stream)))
    a._sync_step(s)


def deferred_update(a: Arena, grads: SparseGrads, *, want_touched: bool = True, stream=None,
                    check_invariants: bool = True):
    """deferred_update (adam.hpp:211-238); returns the touched ids (ascending) when asked."""
    s = a.c_struct()
    g = grads.c_struct()
    dev = a.counter.device
    touched = torch.empty(max(a.count, 1), dtype=torch.int32, device=dev) if want_touched else None
    tcount = torch.zeros(1, dtype=torch.int64, device=dev)
    check(lib().gss_deferred_update(C.byref(s), C.byref(g), _ptr(touched), _ptr(tcount), _stream(stream)))
    if check_invariants:
        check(lib().gss_arena_check(C.byref(s), _stream(stream)))
    a._sync_step(s)
    if want_touched:
        return touched[: int(tcount.item())]
    return tcount


def restore_view(a: Arena, ids: torch.Tensor, pending: Optional[SparseGrads], out: Optional[torch.Tensor] = None,
                 stream=None) -> torch.Tensor:
    """restore_view (adam.hpp:252-289): pure read; arena untouched."""
    n = int(ids.numel())
    if out is None:
        out = torch.empty((max(n, 1), a.dim), dtype=torch.float32, device=a.counter.device)[:n]
    s = a.c_struct()
    pg = pending.c_struct() if pending is not None else None
    check(lib().gss_restore_view(C.byref(s), _ptr(ids) if n else None, n, None,
                                 C.byref(pg) if pg is not None else None, _ptr(out) if n else None, _stream(stream)))
    return out


def set_host_chunk_bytes(nbytes: int) -> None:
    """Chunk size of the staged host-tier passes (ForwardStage chunks, store.hpp:204-213)."""
    check(lib().gss_set_host_chunk_bytes(int(nbytes)))


def flush_deferred(a: Arena, stream=None) -> None:
    s = a.c_struct()
    check(lib().gss_flush_deferred(C.byref(s), _stream(stream)))


# ---------------------------------------------------------------------------------------------
# Rasterizer

@dataclass
class RenderScene:
    """RenderScene (render.hpp:70-77): ids ascending; geo rows by global id; nongeo rows compact
    (slot-indexed, the forwarded slice) or by id."""

    ids: torch.Tensor
    geo: torch.Tensor
    nongeo: torch.Tensor
    nongeo_compact: bool = False
    geo_stride: int = K_GEO_DIM
    nongeo_stride: int = K_NONGEO_DIM
    slot_map: Optional[torch.Tensor] = None
    sh_degree: int = 3
    background: tuple = (0.0, 0.0, 0.0)
    low_pass: float = K_LOW_PASS

    def c_struct(self) -> GssRenderScene:
        s = GssRenderScene()
        s.ids = _ptr(self.ids) if self.ids.numel() else None
        s.count = int(self.ids.numel())
        s.count_dev = None
        s.geo, s.geo_stride = _ptr(self.geo), int(self.geo_stride)
        s.nongeo, s.nongeo_stride = _ptr(self.nongeo), int(self.nongeo_stride)
        s.nongeo_compact = 1 if self.nongeo_compact else 0
        s.slot_map = _ptr(self.slot_map)
        s.sh_degree = int(self.sh_degree)
        for i in range(3):
            s.background[i] = float(self.background[i])
        s.low_pass = float(self.low_pass)
        return s


class _Ctx:
    def __init__(self):
        self.h = lib().gss_render_ctx_create()
        if not self.h:
            check(1)

    def __del__(self):
        h = getattr(self, "h", None)
        if h:
            try:
                torch.cuda.synchronize()
            except Exception:
                pass
            lib().gss_render_ctx_destroy(h)
            self.h = None


@dataclass
class RenderResult:
    """RenderResult (render.hpp:284-289) with the aux kept on the device inside `ctx`."""

    image: torch.Tensor  # ph x pw x 3
    final_T: torch.Tensor  # ph x pw
    n_contrib: torch.Tensor  # ph x pw (used contributions per pixel, aux.len)
    px0: int
    py0: int
    pw: int
    ph: int
    visible: int
    instances: int
    ctx: _Ctx
    scene: RenderScene
    loss: Optional[torch.Tensor] = None
    d_img: Optional[torch.Tensor] = None


def rasterize_forward(sc: RenderScene, cam: GssCamera, vp: GssViewport, *, gt: Optional[torch.Tensor] = None,
                      normalizer: int = 0, ctx: Optional[_Ctx] = None, stream=None) -> RenderResult:
    """rasterize_forward (render.hpp:384-464); with gt (full camera image) the L1 loss and its
    gradient (compute_loss_l1, render.hpp:497-511) are fused into the composite kernel."""
    ctx = ctx or _Ctx()
    dev = sc.geo.device
    import math
    px0 = max(int(math.ceil(float(np.float32(vp.x0)) - 0.5)), 0)
    py0 = max(int(math.ceil(float(np.float32(vp.y0)) - 0.5)), 0)
    pw = max(0, int(math.ceil(float(np.float32(vp.x1)) - 0.5)) - px0)
    ph = max(0, int(math.ceil(float(np.float32(vp.y1)) - 0.5)) - py0)
    image = torch.empty((ph, pw, 3), dtype=torch.float32, device=dev)
    fT = torch.empty((ph, pw), dtype=torch.float32, device=dev)
    nc = torch.empty((ph, pw), dtype=torch.int32, device=dev)
    loss = d_img = None
    if gt is not None:
        d_img = torch.empty((ph, pw, 3), dtype=torch.float32, device=dev)
        loss = torch.zeros(1, dtype=torch.float32, device=dev)
    meta = (C.c_int64 * 6)()
    s = sc.c_struct()
    check(lib().gss_rasterize_forward(ctx.h, C.byref(s), C.byref(cam), C.byref(vp), _ptr(image),
                                      _ptr(gt), int(normalizer), _ptr(d_img), _ptr(loss), _ptr(fT), _ptr(nc), meta,
                                      _stream(stream)))
    return RenderResult(image, fT, nc, int(meta[0]), int(meta[1]), int(meta[2]), int(meta[3]), int(meta[4]),
                        int(meta[5]), ctx, sc, loss, d_img)


def compute_loss_l1(img: torch.Tensor, gt: torch.Tensor, normalizer: int = 0, stream=None):
    """compute_loss_l1 (render.hpp:497-511): returns (loss device scalar, d_img)."""
    if img.shape != gt.shape:
        raise ConfigError(2, "compute_loss_l1: image and ground-truth shapes differ")
    d = torch.empty_like(img)
    loss = torch.zeros(1, dtype=torch.float32, device=img.device)
    check(lib().gss_loss_l1(_ptr(img), _ptr(gt), img.numel(), int(normalizer), _ptr(d), _ptr(loss), _stream(stream)))
    return loss, d


@dataclass
class GradBuffer:
    """GradBuffer (render.hpp:516-524)."""

    ids: torch.Tensor
    rows: torch.Tensor  # V x 59
    mean2d: torch.Tensor  # V x 2


def rasterize_backward(sc: RenderScene, cam: GssCamera, fw: RenderResult, d_img: torch.Tensor,
                       stream=None) -> GradBuffer:
    """rasterize_backward (render.hpp:526-640), deterministic."""
    V = int(sc.ids.numel())
    dev = sc.geo.device
    rows = torch.zeros((max(V, 1), K_PARAM_DIM), dtype=torch.float32, device=dev)
    m2d = torch.zeros((max(V, 1), 2), dtype=torch.float32, device=dev)
    check(lib().gss_rasterize_backward(fw.ctx.h, _ptr(d_img), _ptr(rows), K_PARAM_DIM, rows.data_ptr() + 40,
                                       K_PARAM_DIM, _ptr(m2d), _stream(stream)))
    return GradBuffer(sc.ids, rows[:V], m2d[:V])


# ---------------------------------------------------------------------------------------------
# Split-phase rasterizer (image-parallel rendering across GPUs; include/gss_b200.h)

SPLAT_RECORD_BYTES = 64


def project(sc: RenderScene, cam: GssCamera, vp: GssViewport, stream=None) -> torch.Tensor:
    """project_all (render.hpp:361-380): one 64-byte splat record per visible slot (uint8 [V, 64])."""
    V = int(sc.ids.numel())
    recs = torch.empty((max(V, 1), SPLAT_RECORD_BYTES), dtype=torch.uint8, device=sc.geo.device)[:V]
    s = sc.c_struct()
    check(lib().gss_project(C.byref(s), C.byref(cam), C.byref(vp), _ptr(recs) if V else None, _stream(stream)))
    return recs


def route_strips(recs: torch.Tensor, strip_x: Sequence[int], stream=None):
    """Slots (ascending) whose pixel box touches each column strip [strip_x[k], strip_x[k+1]).
    Returns (dest_slots [nstrips, V] int32 device, counts host list)."""
    V = int(recs.shape[0])
    k = len(strip_x) - 1
    sx = np.ascontiguousarray(np.asarray(strip_x, np.int32))
    slots = torch.empty((k, max(V, 1)), dtype=torch.int32, device=recs.device)
    counts = torch.zeros(k, dtype=torch.int64, device=recs.device)
    check(lib().gss_route_strips(_ptr(recs) if V else None, V, sx.ctypes.data, k, _ptr(slots), _ptr(counts),
                                 _stream(stream)))
    return slots, [int(c) for c in counts.cpu().tolist()]


def gather_records(recs: torch.Tensor, slots: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None):
    n = int(slots.numel())
    if out is None:
        out = torch.empty((n, SPLAT_RECORD_BYTES), dtype=torch.uint8, device=recs.device)
    check(lib().gss_gather_records(_ptr(recs), _ptr(slots), n, _ptr(out), _stream(stream)))
    return out


def scatter_add_rows(src: torch.Tensor, slots: torch.Tensor, dst: torch.Tensor, stream=None) -> None:
    n = int(slots.numel())
    check(lib().gss_scatter_add_rows(_ptr(src), _ptr(slots), n, int(dst.shape[1]), _ptr(dst), _stream(stream)))


@dataclass
class RecordsResult:
    image: torch.Tensor  # strip window ph x pw x 3
    loss_sum: Optional[torch.Tensor]  # device float64: sum |image - gt| over the window
    d_img: Optional[torch.Tensor]
    px0: int
    py0: int
    pw: int
    ph: int
    count: int
    instances: int
    ctx: "_Ctx"


def rasterize_records_forward(recs: torch.Tensor, cam: GssCamera, vp: GssViewport, *,
                              background=(0.0, 0.0, 0.0), gt: Optional[torch.Tensor] = None, normalizer: int = 0,
                              ctx: Optional["_Ctx"] = None, stream=None) -> RecordsResult:
    """Composite received records on window vp (an image strip); ties in depth follow record order."""
    ctx = ctx or _Ctx()
    dev = recs.device
    import math
    px0 = max(int(math.ceil(float(np.float32(vp.x0)) - 0.5)), 0)
    py0 = max(int(math.ceil(float(np.float32(vp.y0)) - 0.5)), 0)
    pw = max(0, int(math.ceil(float(np.float32(vp.x1)) - 0.5)) - px0)
    ph = max(0, int(math.ceil(float(np.float32(vp.y1)) - 0.5)) - py0)
    image = torch.empty((ph, pw, 3), dtype=torch.float32, device=dev)
    d_img = loss = lsum = None
    if gt is not None:
        d_img = torch.empty((ph, pw, 3), dtype=torch.float32, device=dev)
        loss = torch.zeros(1, dtype=torch.float32, device=dev)
        lsum = torch.zeros(1, dtype=torch.float64, device=dev)
    bg = np.asarray(background, np.float32)
    meta = (C.c_int64 * 6)()
    n = int(recs.shape[0])
    check(lib().gss_rasterize_records_forward(ctx.h, _ptr(recs) if n else None, n, C.byref(cam), C.byref(vp),
                                              bg.ctypes.data, _ptr(image), _ptr(gt), int(normalizer), _ptr(d_img),
                                              _ptr(loss), _ptr(lsum), None, None, meta, _stream(stream)))
    return RecordsResult(image, lsum, d_img, int(meta[0]), int(meta[1]), int(meta[2]), int(meta[3]), n,
                         int(meta[5]), ctx)


def rasterize_records_backward(fw: RecordsResult, d_img: torch.Tensor, stream=None) -> torch.Tensor:
    """Per-record 9-float screen-space gradient sums [count, 9]."""
    sums = torch.zeros((max(fw.count, 1), 9), dtype=torch.float32, device=d_img.device)[: fw.count]
    check(lib().gss_rasterize_records_backward(fw.ctx.h, _ptr(d_img), _ptr(sums) if fw.count else None,
                                               _stream(stream)))
    return sums


def chain_backward(sc: RenderScene, cam: GssCamera, recs: torch.Tensor, sums: torch.Tensor, stream=None) -> GradBuffer:
    """render.hpp:600-638 per slot from the strip-summed screen-space gradients."""
    V = int(sc.ids.numel())
    dev = sc.geo.device
    rows = torch.zeros((max(V, 1), K_PARAM_DIM), dtype=torch.float32, device=dev)
    m2d = torch.zeros((max(V, 1), 2), dtype=torch.float32, device=dev)
    s = sc.c_struct()
    check(lib().gss_chain_backward(C.byref(s), C.byref(cam), _ptr(recs) if V else None, _ptr(sums) if V else None,
                                   _ptr(rows), K_PARAM_DIM, rows.data_ptr() + 40, K_PARAM_DIM, _ptr(m2d),
                                   _stream(stream)))
    return GradBuffer(sc.ids, rows[:V], m2d[:V])


# ---------------------------------------------------------------------------------------------
# Scenes (synth.hpp:13-159) — input generation

@dataclass
class SynthConfig:
    seed: int = 1
    n: int = 300
    cams: int = 32
    width: int = 64
    height: int = 64
    sh_degree: int = 3
    box: float = 1.0
    radius_min: float = 0.3
    radius_max: float = 3.0
    fov_deg: float = 30.0
    fov_ramp: float = 0.4
    target_jitter: float = 1.1
    near_plane: float = 0.05
    far_plane: float = 100.0
    scale_min: float = 0.025
    scale_max: float = 0.07
    scale_aniso: float = 0.5
    opacity_min: float = 0.35
    opacity_max: float = 0.9
    sh_rest_noise: float = 0.12

    @staticmethod
    def low_use(n: int, cams: int, img: int, seed: int) -> "SynthConfig":  # synth.hpp:33-47
        return SynthConfig(seed=seed, n=n, cams=cams, width=img, height=img, radius_min=0.3, radius_max=0.65,
                           fov_deg=20.0, fov_ramp=0.7, target_jitter=1.2, scale_min=0.02, scale_max=0.05)

    def cfg_array(self) -> np.ndarray:
        return np.array([self.box, self.radius_min, self.radius_max, self.fov_deg, self.fov_ramp, self.target_jitter,
                         self.near_plane, self.far_plane, self.scale_min, self.scale_max, self.scale_aniso,
                         self.opacity_min, self.opacity_max, self.sh_rest_noise], dtype=np.float64)


def synth_scene_params(cfg: SynthConfig):
    """Truth rows (n x 59, numpy) + cameras (list of GssCamera), bit-identical to synth_scene."""
    rows = np.zeros((max(cfg.n, 1), K_PARAM_DIM), dtype=np.float32)
    cams = (GssCamera * max(cfg.cams, 1))()
    arr = cfg.cfg_array()
    check(lib().gss_synth_scene(int(cfg.seed), int(cfg.n), int(cfg.cams), int(cfg.width), int(cfg.height),
                                int(cfg.sh_degree), arr.ctypes.data, rows.ctypes.data, C.addressof(cams)))
    return rows[: cfg.n], [cams[i] for i in range(cfg.cams)]


def init_gaussians(positions: np.ndarray, colors: Optional[np.ndarray] = None, knn: int = 3,
                   min_knn_dist: float = 0.01, init_opacity: float = 0.1) -> np.ndarray:
    """init_gaussians (scene.hpp:146-195) with the exact O(M^2) kNN on the device: rows m x 59."""
    pos = np.ascontiguousarray(positions, np.float32).reshape(-1, 3)
    m = pos.shape[0]
    col = None if colors is None else np.ascontiguousarray(colors, np.float32).reshape(-1, 3)
    rows = np.zeros((max(m, 1), K_PARAM_DIM), np.float32)
    check(lib().gss_init_gaussians(pos.ctypes.data, None if col is None else col.ctypes.data, m, int(knn),
                                   float(min_knn_dist), float(init_opacity), rows.ctypes.data))
    return rows[:m]


class PointCloud:
    """PointCloud (scene.hpp:128-133): positions m x 3, colors m x 3 in [0, 1] or None."""

    def __init__(self, positions, colors=None):
        self.positions = positions
        self.colors = colors

    def size(self) -> int:
        return int(self.positions.shape[0])


def load_ply(path, device: Optional[torch.device] = None) -> PointCloud:
    """load_ply (ply.hpp:10-14, ply.cpp:53-199): ASCII or binary little-endian PLY with x,y,z
    (+ red/green/blue or r/g/b). Binary bodies are decoded on the GPU; `device` keeps the result
    there (torch tensors) instead of returning numpy arrays. Raises ParseError like the reference."""
    h = C.c_void_p()
    m = C.c_int64()
    hc = C.c_int32()
    check(lib().gss_ply_open(str(path).encode(), C.byref(h), C.byref(m), C.byref(hc)))
    try:
        n = int(m.value)
        if device is not None:
            pos = torch.empty((n, 3), dtype=torch.float32, device=device)
            col = torch.empty((n, 3), dtype=torch.float32, device=device) if hc.value else None
            check(lib().gss_ply_read(h, pos.data_ptr(), None if col is None else col.data_ptr(),
                                     torch.cuda.current_stream(device).cuda_stream))
        else:
            pos = np.empty((n, 3), np.float32)
            col = np.empty((n, 3), np.float32) if hc.value else None
            check(lib().gss_ply_read(h, pos.ctypes.data, None if col is None else col.ctypes.data, None))
    finally:
        lib().gss_ply_close(h)
    return PointCloud(pos, col)


def save_ply(path, pc: PointCloud, binary: bool = True) -> None:
    """save_ply (ply.hpp:16-17, ply.cpp:201-225)."""
    pos = np.ascontiguousarray(pc.positions, np.float32).reshape(-1, 3)
    col = None if pc.colors is None else np.ascontiguousarray(pc.colors, np.float32).reshape(-1, 3)
    check(lib().gss_save_ply(str(path).encode(), pos.ctypes.data, None if col is None else col.ctypes.data,
                             pos.shape[0], 1 if binary else 0))


def init_from_ply(path, knn: int = 3, min_knn_dist: float = 0.01, init_opacity: float = 0.1) -> np.ndarray:
    """PLY -> init_gaussians rows (m x 59): the real-scene entry of the training path
    (trainer.hpp's scene setup: load_ply then init_gaussians)."""
    pc = load_ply(path)
    return init_gaussians(pc.positions, pc.colors, knn, min_knn_dist, init_opacity)


def render_view(rows: torch.Tensor, cam: GssCamera, sh_degree: int, background=(0.0, 0.0, 0.0)) -> torch.Tensor:
    """render_view (synth.hpp:81-94) on the device: cull + rasterize over a full viewport."""
    geo = rows[:, :K_GEO_DIM].contiguous()
    ng = rows[:, K_GEO_DIM:].contiguous()
    vp = viewport_full(cam.width, cam.height)
    ids = frustum_cull(geo, geo.shape[0], cam, vp)
    sc = RenderScene(ids=ids, geo=geo, nongeo=ng, nongeo_compact=False, sh_degree=sh_degree, background=background)
    return rasterize_forward(sc, cam, vp).image


# ---------------------------------------------------------------------------------------------
# Offload engine

@dataclass
class OptimConfig:
    """OptimConfig (store.hpp:110-145)."""

    lr_mean: float = 1.6e-4
    lr_scale: float = 5e-3
    lr_quat: float = 1e-3
    lr_opacity: float = 5e-2
    lr_sh: float = 2.5e-3
    sh_rest_divisor: float = 20.0
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    defer_max: int = 15
    geo_defer_max: int = 0
    scene_extent: float = 1.0

    def geo_groups(self):
        hp = lambda lr: Hyperparams(lr, self.beta1, self.beta2, self.eps)  # noqa: E731
        return [GroupSpec("mean", 0, 3, hp(self.lr_mean * self.scene_extent)), GroupSpec("scale", 3, 3, hp(self.lr_scale)),
                GroupSpec("quat", 6, 4, hp(self.lr_quat))]

    def nongeo_groups(self):
        hp = lambda lr: Hyperparams(lr, self.beta1, self.beta2, self.eps)  # noqa: E731
        return [GroupSpec("opacity", 0, 1, hp(self.lr_opacity)), GroupSpec("sh_dc", 1, 3, hp(self.lr_sh)),
                GroupSpec("sh_rest", 4, 45, hp(self.lr_sh / self.sh_rest_divisor))]

    def full_groups(self):
        hp = lambda lr: Hyperparams(lr, self.beta1, self.beta2, self.eps)  # noqa: E731
        return [GroupSpec("mean", 0, 3, hp(self.lr_mean * self.scene_extent)), GroupSpec("scale", 3, 3, hp(self.lr_scale)),
                GroupSpec("quat", 6, 4, hp(self.lr_quat)), GroupSpec("opacity", 10, 1, hp(self.lr_opacity)),
                GroupSpec("sh_dc", 11, 3, hp(self.lr_sh)),
                GroupSpec("sh_rest", 14, 45, hp(self.lr_sh / self.sh_rest_divisor))]


@dataclass
class DensifyConfig:
    """DensifyConfig (trainer.hpp:32-47) thresholds."""

    grad_threshold: float = 2e-4
    percent_dense: float = 0.01
    opacity_prune: float = 0.005
    split_scale_divisor: float = 1.6

    def c_struct(self) -> GssDensifyConfig:
        return GssDensifyConfig(self.grad_threshold, self.percent_dense, self.opacity_prune, self.split_scale_divisor)


def plan_densify(rows: torch.Tensor, accum_norm: torch.Tensor, accum_cnt: torch.Tensor, cfg: DensifyConfig,
                 extent: float, seed: int, stream=None):
    """plan_densify (trainer.hpp:166-213) on a device snapshot (n x 59): (survivors ascending,
    child rows k x 59, counts dict)."""
    n = int(rows.shape[0])
    dev = rows.device
    surv = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    kids = torch.empty((max(2 * n, 1), K_PARAM_DIM), dtype=torch.float32, device=dev)
    counts = np.zeros(5, np.int64)
    c = cfg.c_struct()
    check(lib().gss_plan_densify(_ptr(rows), n, _ptr(accum_norm), _ptr(accum_cnt), C.byref(c), float(extent),
                                 int(seed) & 0xFFFFFFFFFFFFFFFF, _ptr(surv), _ptr(kids), counts.ctypes.data,
                                 _stream(stream)))
    torch.cuda.current_stream().synchronize()
    k = dict(zip(("survivors", "children", "clones", "splits", "pruned"), counts.tolist()))
    return surv[: k["survivors"]], kids[: k["children"]], k


class OffloadEngine:
    """OffloadEngine (engine.hpp:55-192) on the B200: two CUDA streams replace the two workers."""

    def __init__(self, init_rows: np.ndarray, cams: Sequence[GssCamera], gts: Optional[np.ndarray],
                 optim: OptimConfig = OptimConfig(), *, pipelined: bool = True, sh_degree: int = 3,
                 sh_warmup_step: int = 0, background=(0.0, 0.0, 0.0), low_pass: float = K_LOW_PASS,
                 nongeo_on_host: bool = False, splits=None):
        cfg = GssEngineConfig()
        lib().gss_engine_config_default(C.byref(cfg))
        for k in ("lr_mean", "lr_scale", "lr_quat", "lr_opacity", "lr_sh", "sh_rest_divisor", "beta1", "beta2", "eps",
                  "scene_extent", "defer_max", "geo_defer_max"):
            setattr(cfg, k, getattr(optim, k))
        cfg.pipelined = 1 if pipelined else 0
        cfg.sh_degree, cfg.sh_warmup_step = int(sh_degree), int(sh_warmup_step)
        for i in range(3):
            cfg.background[i] = float(background[i])
        cfg.low_pass = float(low_pass)
        cfg.nongeo_on_host = 1 if nongeo_on_host else 0
        rows = np.ascontiguousarray(init_rows, dtype=np.float32)
        self.n = rows.shape[0]
        self.ncams = len(cams)
        cam_arr = (GssCamera * max(len(cams), 1))(*cams)
        self._gts = None if gts is None else np.ascontiguousarray(gts, dtype=np.float32)
        self.h = lib().gss_engine_create(self.n, rows.ctypes.data, len(cams), C.addressof(cam_arr),
                                         None if self._gts is None else self._gts.ctypes.data, C.byref(cfg))
        if not self.h:
            check(int(1) if "device" in lib().gss_last_error().decode() else 2)
        if splits is not None:
            self.set_splits(splits)

    def set_splits(self, splits):
        """SplitTable (splitter.hpp:12-23; OffloadEngine constructor, engine.hpp:62-68): one
        (split, column) pair per stored camera — or SplitEntry-like objects with .split/.column, or
        the dicts of evalsplit.compute_split_points. run() renders split cameras as two sub-passes."""
        flags = np.zeros(len(splits), np.int32)
        cols = np.zeros(len(splits), np.int32)
        for i, e in enumerate(splits):
            if isinstance(e, dict):
                sp, col = e["split"], e["column"]
            elif hasattr(e, "split"):
                sp, col = e.split, e.column
            else:
                sp, col = e
            flags[i], cols[i] = int(bool(sp)), int(col)
        check(lib().gss_engine_set_splits(self.h, len(splits), flags.ctypes.data, cols.ctypes.data))

    def close(self):
        if getattr(self, "h", None):
            lib().gss_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def run(self, n: int):
        losses = np.zeros(max(n, 1), np.float32)
        valid = np.zeros(max(n, 1), np.int32)
        check(lib().gss_engine_run(self.h, int(n), losses.ctypes.data, valid.ctypes.data))
        return losses[:n], valid[:n]

    def step(self, cam: GssCamera, gt_host: np.ndarray):
        loss = C.c_float(0)
        valid = C.c_int32(0)
        gt = gt_host if isinstance(gt_host, np.ndarray) else gt_host.numpy()
        gt = np.ascontiguousarray(gt, dtype=np.float32)
        if gt.size != cam.width * cam.height * 3:
            raise ConfigError(2, "step: gt_host must hold height*width*3 floats")
        check(lib().gss_engine_step(self.h, C.byref(cam), gt.ctypes.data, C.byref(loss), C.byref(valid)))
        return float(loss.value), int(valid.value)

    def step_async(self, cam: GssCamera, gt_host, loss_out) -> int:
        """gss_engine_step_async: enqueue one iteration and return its valid count. gt_host and
        loss_out are pinned host torch tensors (loss_out a float32 element, e.g. losses[i:i+1]);
        both are owned by the step until drain()."""
        for t in (gt_host, loss_out):
            if not (isinstance(t, torch.Tensor) and t.is_pinned() and t.is_contiguous()):
                raise ValueError("step_async: gt_host / loss_out must be contiguous pinned host tensors")
        if gt_host.dtype != torch.float32 or loss_out.dtype != torch.float32 or loss_out.numel() < 1:
            raise ValueError("step_async: float32 tensors required")
        if gt_host.numel() != cam.width * cam.height * 3:
            raise ValueError("step_async: gt_host must hold height*width*3 floats")
        valid = C.c_int32(0)
        check(lib().gss_engine_step_async(self.h, C.byref(cam), gt_host.data_ptr(), loss_out.data_ptr(),
                                          C.byref(valid)))
        return int(valid.value)

    def drain(self):
        check(lib().gss_engine_drain(self.h))

    def snapshot(self) -> np.ndarray:
        out = np.zeros((max(self.n, 1), K_PARAM_DIM), np.float32)
        check(lib().gss_engine_snapshot(self.h, out.ctypes.data))
        return out[: self.n]

    def state(self):
        n = max(self.n, 1)
        geo_w = np.zeros((n, K_GEO_DIM), np.float32)
        ng_w = np.zeros((n, K_NONGEO_DIM), np.float32)
        ng_m = np.zeros((n, K_NONGEO_DIM), np.float32)
        ng_v = np.zeros((n, K_NONGEO_DIM), np.float32)
        cnt = np.zeros(n, np.uint8)
        steps = np.zeros(2, np.int64)
        check(lib().gss_engine_state(self.h, geo_w.ctypes.data, ng_w.ctypes.data, ng_m.ctypes.data, ng_v.ctypes.data,
                                     cnt.ctypes.data, steps.ctypes.data))
        k = self.n
        return dict(geo_w=geo_w[:k], ng_w=ng_w[:k], ng_m=ng_m[:k], ng_v=ng_v[:k], ng_counter=cnt[:k],
                    geo_step=int(steps[0]), ng_step=int(steps[1]))

    def accum(self):
        norm = np.zeros(max(self.n, 1), np.float64)
        cnt = np.zeros(max(self.n, 1), np.int32)
        check(lib().gss_engine_accum(self.h, norm.ctypes.data, cnt.ctypes.data))
        return norm[: self.n], cnt[: self.n]

    def stage_ms(self):
        out = np.zeros(6, np.float64)
        check(lib().gss_engine_stage_ms(self.h, out.ctypes.data))
        return dict(zip(("cull", "forward_params", "render", "geo_update", "handoff", "lazy_update"), out.tolist()))

    def launches(self) -> int:
        return int(lib().gss_engine_launches(self.h))

    TIMELINE_STAGES = ("cull", "forward_params", "render", "geo_update", "handoff", "lazy_update")

    def timeline_enable(self, on: bool = True) -> None:
        """Per-iteration stage timeline (engine.hpp:22-28): rows from now on, times from now."""
        check(lib().gss_engine_timeline_enable(self.h, 1 if on else 0))

    def timeline(self):
        """TimelineRow list: dicts with iteration, stage, worker (0 device, 1 host tier), t0_ns,
        t1_ns, bytes."""
        n = int(lib().gss_engine_timeline(self.h, None, 0))
        if n < 0:
            check(-n)
        rows = np.zeros((max(n, 1), 5), np.int64)  # gss_timeline_row: 40 bytes
        m = int(lib().gss_engine_timeline(self.h, rows.ctypes.data, n))
        if m < 0:
            check(-m)
        out = []
        for r in rows[:n]:
            it, st = int(r[0]) & 0xFFFFFFFF, int(r[0]) >> 32
            wk = int(r[1]) & 0xFFFFFFFF
            out.append({"iteration": it if it < 2 ** 31 else it - 2 ** 32, "stage": self.TIMELINE_STAGES[st],
                        "worker": wk, "t0_ns": int(r[2]), "t1_ns": int(r[3]), "bytes": int(r[4]) & (2 ** 64 - 1)})
        return out

    def stage_delays(self, ns) -> None:
        """Test instrumentation: device-side sleeps (ns) at each stage start, cycling (the
        reference's EngineConfig::stage_hook delays). Empty list disables."""
        arr = np.ascontiguousarray(np.asarray(ns, np.uint32))
        check(lib().gss_engine_stage_delays(self.h, arr.ctypes.data if arr.size else None, int(arr.size)))

    def kernel_timing(self, on: bool = True) -> None:
        """CUDA events around every composite / sweep kernel launch (see kernel_times)."""
        check(lib().gss_engine_kernel_timing(self.h, 1 if on else 0))

    def kernel_times(self):
        """Drains; {composite_ms, sweep_ms, composite_launches, sweep_launches, contribs} since the
        last call (contribs = contributions composited = useful backward contributions)."""
        ms = np.zeros(6, np.float64)
        n = np.zeros(6, np.int64)
        c = C.c_uint64()
        check(lib().gss_engine_render_times(self.h, ms.ctypes.data, n.ctypes.data, C.byref(c)))
        out = {"composite_ms": float(ms[0]), "sweep_ms": float(ms[1]), "composite_launches": int(n[0]),
               "sweep_launches": int(n[1]), "contribs": int(c.value)}
        for i, k in ((2, "geometry"), (3, "colour"), (4, "slot_sums"), (5, "chain")):
            out[f"{k}_ms"] = float(ms[i])
            out[f"{k}_launches"] = int(n[i])
        return out

    def densify(self, cfg: DensifyConfig, extent: float, seed: int):
        """A densification event (trainer.hpp:578-591): snapshot, plan_densify, apply_densify."""
        counts = np.zeros(6, np.int64)
        c = cfg.c_struct()
        check(lib().gss_engine_densify(self.h, C.byref(c), float(extent), int(seed) & 0xFFFFFFFFFFFFFFFF,
                                       counts.ctypes.data))
        self.n = int(counts[5])
        return dict(zip(("survivors", "children", "clones", "splits", "pruned", "n"), counts.tolist()))


def launch_count() -> int:
    return int(lib().gss_launch_count())
