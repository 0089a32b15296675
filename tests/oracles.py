"""Test-only ctypes bindings to the two CPU checkers under oracle/_ref/:

* ``libgss_ref.so``   — the UNMODIFIED reference headers behind oracle/ref_shim.cpp (the reference
  path itself, built here from /root/reference; shipped to the GPU box as a prebuilt .so);
* ``libgss_oracle.so`` — the C restatement oracle/gss_oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py's reference/cpu_baseline legs import this.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_SO = ROOT / "oracle" / "_ref" / "libgss_ref.so"
ORC_SO = ROOT / "oracle" / "_ref" / "libgss_oracle.so"

P, I64, I32, F32, F64 = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_double


def _p(a):
    return None if a is None else a.ctypes.data


_ref = None
_orc = None


def ref():
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            return None
        l = C.CDLL(str(REF_SO))
        sig = {
            "ref_expf": (F32, [F32]),
            "ref_frustum_cull": (C.c_int, [P, C.c_int, C.c_int, P, P, F32, P]),
            "ref_project_geo": (None, [P, P, F32, P]),
            "ref_render": (C.c_int, [C.c_int, P, P, C.c_int, P, C.c_int, C.c_int, P, P, P, P, I64, P, C.c_int,
                                     P, P, P, P, P, P, P, P, P]),
            "ref_loss_l1": (C.c_int, [P, P, C.c_int, C.c_int, I64, P, P]),
            "ref_build_luts": (None, [F64, F64, F64, F64, I64, C.c_int, P, P, P, P, P, P]),
            "ref_arena_new": (P, [C.c_int, C.c_int, C.c_int, P, P, P, F64, F64, F64, C.c_int, P]),
            "ref_arena_free": (None, [P]),
            "ref_arena_ptrs": (None, [P, P, P, P, P, P]),
            "ref_arena_access": (None, [P, P]),
            "ref_adam_step_dense": (C.c_int, [P, P]),
            "ref_deferred_update": (I64, [P, C.c_int, P, P, C.c_int, C.c_int, P]),
            "ref_restore_view": (C.c_int, [P, C.c_int, P, C.c_int, C.c_int, P, P, C.c_int, C.c_int, P]),
            "ref_flush_deferred": (None, [P]),
            "ref_check_counters": (C.c_int, [P]),
            "ref_optim_bench": (None, [C.c_int, C.c_int, C.c_int, F64, C.c_int, C.c_uint64, P]),
            "ref_synth_scene": (None, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P, P, P]),
            "ref_look_at_camera": (None, [P, P, F32, F32, C.c_int, C.c_int, F32, F32, P]),
            "ref_engine_new": (P, [C.c_int, P, C.c_int, P, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P]),
            "ref_engine_new_split": (P, [C.c_int, P, C.c_int, P, P, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P,
                                         P, P]),
            "ref_engine_free": (None, [P]),
            "ref_engine_run": (C.c_int, [P, C.c_int, P, P]),
            "ref_engine_snapshot": (None, [P, P]),
            "ref_engine_state": (None, [P, P, P, P, P, P, P]),
            "ref_engine_accum": (None, [P, P, P]),
            "ref_engine_stage_ns": (None, [P, P]),
            "ref_plan_densify": (None, [C.c_int, P, P, P, P, F64, C.c_uint64, P, P, P]),
            "ref_engine_densify": (C.c_int, [P, P, F64, C.c_uint64, P]),
            "ref_compute_split_points": (None, [P, C.c_int, C.c_int, P, F64, P, P]),
            "ref_psnr_over_views": (F64, [C.c_int, P, C.c_int, P, P, C.c_int, P]),
            "ref_init_gaussians": (C.c_int, [P, P, C.c_int, C.c_int, F64, F64, P]),
            "ref_synth_scene_nogt": (None, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, P, P, P]),
            "ref_render_view_rows": (None, [C.c_int, P, P, C.c_int, C.c_int, P]),
            "ref_load_ply": (C.c_int, [C.c_char_p, I64, P, P, P, P, C.c_char_p, C.c_int]),
            "ref_save_ply": (C.c_int, [C.c_char_p, P, P, C.c_int, C.c_int]),
        }
        for k, (r, a) in sig.items():
            f = getattr(l, k)
            f.restype, f.argtypes = r, a
        _ref = l
    return _ref


def orc():
    global _orc
    if _orc is None:
        if not ORC_SO.exists():
            return None
        l = C.CDLL(str(ORC_SO))
        sig = {
            "orc_expf": (F32, [F32]),
            "orc_project_geo": (None, [P, P, F32, P]),
            "orc_frustum_cull": (I64, [P, I64, I64, P, P, F32, P]),
            "orc_build_luts": (None, [F64, F64, F64, F64, I64, C.c_int, P, P, P, P, P, P]),
            "orc_adam_step_dense": (None, [P, P]),
            "orc_deferred_update": (I64, [P, I64, P, P, I64, C.c_int, P]),
            "orc_restore_view": (None, [P, I64, P, C.c_int, I64, P, P, I64, C.c_int, P]),
            "orc_flush_deferred": (None, [P]),
            "orc_render": (C.c_int, [I64, P, P, I64, P, C.c_int, C.c_int, P, P, P, P, I64, P, P, P, P, P, P, P, P,
                                     P]),
        }
        for k, (r, a) in sig.items():
            f = getattr(l, k)
            f.restype, f.argtypes = r, a
        _orc = l
    return _orc


# ---- camera helpers (80-byte gss_camera as a float32[20] buffer with two int32 slots) -------

def cam_array(rot, trans, fx, fy, cx, cy, w, h, near, far) -> np.ndarray:
    a = np.zeros(20, np.float32)
    a[0:9] = np.asarray(rot, np.float32).reshape(9)
    a[9:12] = np.asarray(trans, np.float32).reshape(3)
    a[12:16] = [fx, fy, cx, cy]
    iv = a.view(np.int32)
    iv[16], iv[17] = int(w), int(h)
    a[18], a[19] = near, far
    return a


def cam_from_struct(c) -> np.ndarray:
    return np.frombuffer(bytes(c), dtype=np.float32).copy()


def cam_wh(cam: np.ndarray):
    iv = cam.view(np.int32)
    return int(iv[16]), int(iv[17])


def basic_cam(w=100, h=100, fx=100.0, near=0.1, far=100.0) -> np.ndarray:
    """test_render.cpp:14-27."""
    return cam_array(np.eye(3), [0, 0, 0], fx, fx, w / 2, h / 2, w, h, near, far)


def look_at(eye, target, fx, fy, w, h, near, far) -> np.ndarray:
    out = np.zeros(20, np.float32)
    e = np.ascontiguousarray(eye, np.float32)
    t = np.ascontiguousarray(target, np.float32)
    ref().ref_look_at_camera(e.ctypes.data, t.ctypes.data, fx, fy, w, h, near, far, out.ctypes.data)
    return out


# ---- reference wrappers ----------------------------------------------------------------------

def ref_cull(geo: np.ndarray, cam: np.ndarray, vp, low_pass=0.3, stride=10) -> np.ndarray:
    geo = np.ascontiguousarray(geo, np.float32)
    n = geo.size // stride
    out = np.zeros(max(n, 1), np.int32)
    vpa = np.asarray(vp, np.float32)
    k = ref().ref_frustum_cull(_p(geo), n, stride, _p(cam), _p(vpa), low_pass, _p(out))
    return out[:k].copy()


def orc_cull(geo: np.ndarray, cam: np.ndarray, vp, low_pass=0.3, stride=10) -> np.ndarray:
    geo = np.ascontiguousarray(geo, np.float32)
    n = geo.size // stride
    out = np.zeros(max(n, 1), np.int32)
    vpa = np.asarray(vp, np.float32)
    k = orc().orc_frustum_cull(_p(geo), n, stride, _p(cam), _p(vpa), low_pass, _p(out))
    return out[:k].copy()


def render(lib_name: str, ids, geo, nongeo, cam, vp, *, compact=False, sh_degree=3, bg=(0, 0, 0), gt=None,
           normalizer=0, d_img=None, geo_stride=10, workers=1):
    """Runs ref_render / orc_render; returns a dict of outputs."""
    ids = np.ascontiguousarray(ids, np.int32)
    geo = np.ascontiguousarray(geo, np.float32)
    nongeo = np.ascontiguousarray(nongeo, np.float32)
    vpa = np.asarray(vp, np.float32)
    bga = np.asarray(bg, np.float32)
    w, h = cam_wh(cam)
    import math
    px0 = max(int(math.ceil(float(vpa[0]) - 0.5)), 0)
    py0 = max(int(math.ceil(float(vpa[2]) - 0.5)), 0)
    pw = max(0, int(math.ceil(float(vpa[1]) - 0.5)) - px0)
    ph = max(0, int(math.ceil(float(vpa[3]) - 0.5)) - py0)
    n = ids.size
    img = np.zeros((max(ph, 1), max(pw, 1), 3), np.float32)
    fT = np.zeros((max(ph, 1), max(pw, 1)), np.float32)
    ln = np.zeros((max(ph, 1), max(pw, 1)), np.int32)
    loss = np.zeros(1, np.float32)
    dimg = np.zeros((max(ph, 1), max(pw, 1), 3), np.float32)
    rows = np.zeros((max(n, 1), 59), np.float32)
    m2d = np.zeros((max(n, 1), 2), np.float32)
    meta = np.zeros(6, np.int64)
    gt_p = None if gt is None else np.ascontiguousarray(gt, np.float32)
    di = None if d_img is None else np.ascontiguousarray(d_img, np.float32)
    if lib_name == "ref":
        st = ref().ref_render(n, _p(ids), _p(geo), geo_stride, _p(nongeo), int(compact), sh_degree, _p(bga), _p(cam),
                              _p(vpa), _p(gt_p), int(normalizer), _p(di), int(workers), _p(img), _p(fT), _p(ln), _p(loss),
                              _p(dimg), _p(rows), _p(m2d), None, _p(meta))
    else:
        st = orc().orc_render(n, _p(ids), _p(geo), geo_stride, _p(nongeo), int(compact), sh_degree, _p(bga), _p(cam),
                              _p(vpa), _p(gt_p), int(normalizer), _p(di), _p(img), _p(fT), _p(ln), _p(loss),
                              _p(dimg), _p(rows), _p(m2d), _p(meta))
    assert st == 0, st
    return dict(image=img[:ph, :pw], final_T=fT[:ph, :pw], len=ln[:ph, :pw], loss=float(loss[0]),
                d_img=dimg[:ph, :pw], rows=rows[:n], mean2d=m2d[:n], contribs=int(meta[4]),
                window=(int(meta[0]), int(meta[1]), int(meta[2]), int(meta[3])))


class RefArena:
    """Reference Arena<float> (adam.hpp:119-159) through the shim; numpy views of its storage."""

    def __init__(self, n, dim, groups, defer_max, b1=0.9, b2=0.999, eps=1e-8):
        col0 = np.array([g[0] for g in groups], np.int32)
        gd = np.array([g[1] for g in groups], np.int32)
        lr = np.array([g[2] for g in groups], np.float64)
        st = C.c_int(0)
        self.h = ref().ref_arena_new(n, dim, len(groups), _p(col0), _p(gd), _p(lr), b1, b2, eps, defer_max,
                                     C.byref(st))
        if not self.h:
            raise ValueError(f"ref arena init failed: status {st.value}")
        self.n, self.dim = n, dim
        ptrs = [C.c_void_p() for _ in range(5)]
        ref().ref_arena_ptrs(self.h, *[C.byref(p) for p in ptrs])
        sz = n * dim

        def view(p, count, dt):
            if count == 0:
                return np.zeros(0, dt)
            buf = (C.c_byte * (count * np.dtype(dt).itemsize)).from_address(p.value)
            return np.frombuffer(buf, dtype=dt)

        self.w = view(ptrs[0], sz, np.float32).reshape(n, dim)
        self.m = view(ptrs[1], sz, np.float32).reshape(n, dim)
        self.v = view(ptrs[2], sz, np.float32).reshape(n, dim)
        self.counter = view(ptrs[3], n, np.uint8)
        self._step = (C.c_int64).from_address(ptrs[4].value)

    @property
    def step(self):
        return self._step.value

    @step.setter
    def step(self, v):
        self._step.value = int(v)

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_arena_free(self.h)
            self.h = None

    def dense(self, grads):
        return ref().ref_adam_step_dense(self.h, _p(grads))

    def deferred(self, ids, rows, stride, col0=0):
        ids = np.ascontiguousarray(ids, np.int32)
        rows = None if rows is None else np.ascontiguousarray(rows, np.float32)
        touched = np.zeros(max(self.n, 1), np.int32)
        k = ref().ref_deferred_update(self.h, ids.size, _p(ids) if ids.size else None,
                                      _p(rows) if rows is not None and rows.size else None, stride, col0, _p(touched))
        if k < 0:
            raise RuntimeError(f"status {-k}")
        return touched[:k].copy()

    def restore(self, ids, pending=None):
        ids = np.ascontiguousarray(ids, np.int32)
        out = np.zeros((max(ids.size, 1), self.dim), np.float32)
        if pending is None:
            st = ref().ref_restore_view(self.h, ids.size, _p(ids), 0, 0, None, None, self.dim, 0, _p(out))
        else:
            pids, prows, pstride, pcol0 = pending
            pids = np.ascontiguousarray(pids, np.int32)
            prows = np.ascontiguousarray(prows, np.float32)
            st = ref().ref_restore_view(self.h, ids.size, _p(ids), 1, pids.size, _p(pids) if pids.size else None,
                                        _p(prows) if prows.size else None, pstride, pcol0, _p(out))
        assert st == 0
        return out[: ids.size]

    def flush(self):
        ref().ref_flush_deferred(self.h)


def ref_luts(lr, t, max_delay, b1=0.9, b2=0.999, eps=1e-8):
    arrs = [np.zeros(max_delay + 1, np.float32) for _ in range(5)]
    sc = np.zeros(5, np.float32)
    ref().ref_build_luts(lr, b1, b2, eps, t, max_delay, *[a.ctypes.data for a in arrs], sc.ctypes.data)
    return arrs, sc


def synth_cfg_array(c) -> np.ndarray:
    return c.cfg_array()


def ref_synth(cfg, with_gt=False):
    rows = np.zeros((max(cfg.n, 1), 59), np.float32)
    cams = np.zeros((max(cfg.cams, 1), 20), np.float32)
    gts = np.zeros((max(cfg.cams, 1), cfg.height, cfg.width, 3), np.float32) if with_gt else None
    arr = cfg.cfg_array()
    ref().ref_synth_scene(cfg.seed, cfg.n, cfg.cams, cfg.width, cfg.height, cfg.sh_degree, arr.ctypes.data,
                          rows.ctypes.data, cams.ctypes.data, None if gts is None else gts.ctypes.data)
    return rows[: cfg.n], cams[: cfg.cams], (None if gts is None else gts[: cfg.cams])


def ref_synth_nogt(cfg):
    """synth_scene (synth.hpp:100-154) without its ground-truth render: (rows n x 59, cams x 20)."""
    rows = np.zeros((max(cfg.n, 1), 59), np.float32)
    cams = np.zeros((max(cfg.cams, 1), 20), np.float32)
    arr = cfg.cfg_array()
    ref().ref_synth_scene_nogt(cfg.seed, cfg.n, cfg.cams, cfg.width, cfg.height, cfg.sh_degree, arr.ctypes.data,
                               rows.ctypes.data, cams.ctypes.data)
    return rows[: cfg.n], cams[: cfg.cams]


def ref_render_view(rows, cam, sh_degree=3, workers=1):
    """render_view (synth.hpp:81-94) of n x 59 rows on the reference renderer."""
    rows = np.ascontiguousarray(rows, np.float32)
    cam = np.ascontiguousarray(cam, np.float32)
    w, h = cam_wh(cam)
    out = np.zeros((h, w, 3), np.float32)
    ref().ref_render_view_rows(rows.shape[0], _p(rows), _p(cam), sh_degree, workers, _p(out))
    return out


OPTIM_DEFAULT = np.array([1.6e-4, 5e-3, 1e-3, 5e-2, 2.5e-3, 20.0, 0.9, 0.999, 1e-8, 1.0], np.float64)


class RefEngine:
    def __init__(self, rows, cams, gts, defer_max=15, geo_defer_max=0, pipelined=False, dense=False, workers=1,
                 sh_degree=3, bg=(0, 0, 0), optim=OPTIM_DEFAULT, splits=None):
        rows = np.ascontiguousarray(rows, np.float32)
        cams = np.ascontiguousarray(cams, np.float32)
        gts = np.ascontiguousarray(gts, np.float32)
        self.n = rows.shape[0]
        flags = (1 if pipelined else 0) | (2 if dense else 0)
        bga = np.asarray(bg, np.float32)
        opt = np.ascontiguousarray(optim, np.float64)
        if splits is None:
            self.h = ref().ref_engine_new(self.n, _p(rows), cams.shape[0], _p(cams), _p(gts), defer_max,
                                          geo_defer_max, flags, workers, sh_degree, _p(bga), _p(opt))
        else:  # (split, column) per camera: the SplitTable of the OffloadEngine constructor
            sp = np.ascontiguousarray([int(bool(a)) for a, _ in splits], np.int32)
            co = np.ascontiguousarray([int(b) for _, b in splits], np.int32)
            self.h = ref().ref_engine_new_split(self.n, _p(rows), cams.shape[0], _p(cams), _p(gts), defer_max,
                                                geo_defer_max, flags, workers, sh_degree, _p(bga), _p(opt),
                                                _p(sp), _p(co))

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_engine_free(self.h)
            self.h = None

    def run(self, n):
        losses = np.zeros(max(n, 1), np.float32)
        valid = np.zeros(max(n, 1), np.int32)
        st = ref().ref_engine_run(self.h, n, _p(losses), _p(valid))
        assert st == 0, st
        return losses[:n], valid[:n]

    def snapshot(self):
        out = np.zeros((max(self.n, 1), 59), np.float32)
        ref().ref_engine_snapshot(self.h, _p(out))
        return out[: self.n]

    def state(self):
        n = max(self.n, 1)
        geo = np.zeros((n, 10), np.float32)
        ngw = np.zeros((n, 49), np.float32)
        ngm = np.zeros((n, 49), np.float32)
        ngv = np.zeros((n, 49), np.float32)
        cnt = np.zeros(n, np.uint8)
        steps = np.zeros(2, np.int64)
        ref().ref_engine_state(self.h, _p(geo), _p(ngw), _p(ngm), _p(ngv), _p(cnt), _p(steps))
        k = self.n
        return dict(geo_w=geo[:k], ng_w=ngw[:k], ng_m=ngm[:k], ng_v=ngv[:k], ng_counter=cnt[:k],
                    geo_step=int(steps[0]), ng_step=int(steps[1]))

    def accum(self):
        norm = np.zeros(max(self.n, 1), np.float64)
        cnt = np.zeros(max(self.n, 1), np.int32)
        ref().ref_engine_accum(self.h, _p(norm), _p(cnt))
        return norm[: self.n], cnt[: self.n]

    def densify(self, dcfg, extent, seed):
        """plan_densify + apply_densify (trainer.hpp:578-591) on the reference engine."""
        counts = np.zeros(5, np.int64)
        st = ref().ref_engine_densify(self.h, _p(np.asarray(dcfg, np.float64)), float(extent), int(seed), _p(counts))
        assert st == 0, st
        self.n = int(counts[0] + counts[1])
        return counts

    def stage_ns(self):
        out = np.zeros(6, np.int64)
        ref().ref_engine_stage_ns(self.h, _p(out))
        return out


# ---- shared generators (mirroring the reference tests' scene builders) -----------------------

def rel_err(a, b):
    """test_util.hpp:17-19."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.maximum(1.0, np.abs(a)), np.abs(b))


def rel_err_floor(a, b, floor):
    """test_util.hpp:22-24."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.abs(a - b) / np.maximum(np.maximum(floor, np.abs(a)), np.abs(b))


class Rng:
    """rng.hpp:11-51 (splitmix64 + Box-Muller), for test input generation."""

    MASK = (1 << 64) - 1

    def __init__(self, seed):
        self.s = seed & self.MASK
        self.spare = None

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & self.MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.MASK
        return z ^ (z >> 31)

    def uniform(self, lo=0.0, hi=1.0):
        u = float(self.next_u64() >> 11) * 2.0 ** -53
        return lo + (hi - lo) * u if (lo, hi) != (0.0, 1.0) else u

    def normal(self):
        import math
        if self.spare is not None:
            s, self.spare = self.spare, None
            return s
        u1 = self.uniform()
        u2 = self.uniform()
        if u1 < 1e-300:
            u1 = 1e-300
        r = math.sqrt(-2.0 * math.log(u1))
        a = 6.283185307179586477 * u2
        self.spare = r * math.sin(a)
        return r * math.cos(a)


def acceptance5_scene(rng: Rng, n=200):
    """acceptance.cpp:215-257: random geometric rows + a look-at camera, 48x40 viewport."""
    import math
    rows = np.zeros((n, 10), np.float32)
    for i in range(n):
        q = [rng.normal() for _ in range(4)]
        qn = math.sqrt(max(sum(c * c for c in q), 1e-12))
        vals = [rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(-4, 8), rng.uniform(-3.5, -0.5),
                rng.uniform(-3.5, -0.5), rng.uniform(-3.5, -0.5), q[0] / qn, q[1] / qn, q[2] / qn, q[3] / qn]
        rows[i] = np.array(vals, np.float64).astype(np.float32)
    eye = np.array([rng.uniform(-2, 2), rng.uniform(-2, 2), rng.uniform(-4, -2)], np.float64).astype(np.float32)
    tgt = np.array([rng.uniform(-0.5, 0.5), rng.uniform(-0.5, 0.5), 0.0], np.float64).astype(np.float32)
    cam = look_at(eye, tgt, 50.0, 50.0, 48, 40, 0.8, 7.0)
    return rows, cam


def check_scene(seed, n, img, sh_degree):
    """test_util.hpp:97-127 (make_check_scene<float>): rows n x 59, camera, gt image."""
    import math
    rng = Rng(seed)
    rows = np.zeros((n, 59), np.float32)
    for i in range(n):
        rows[i, 0] = np.float32(rng.uniform(-0.5, 0.5))
        rows[i, 1] = np.float32(rng.uniform(-0.5, 0.5))
        rows[i, 2] = np.float32(rng.uniform(-0.4, 0.4))
        for a in range(3):
            rows[i, 3 + a] = np.float32(rng.uniform(math.log(0.06), math.log(0.28)))
        q = [rng.normal() for _ in range(4)]
        qn = math.sqrt(max(sum(c * c for c in q), 1e-12))
        for a in range(4):
            rows[i, 6 + a] = np.float32(q[a] / qn)
        p = rng.uniform(0.15, 0.45)
        rows[i, 10] = np.float32(math.log(p) - math.log(1.0 - p))
        for c in range(3):
            rows[i, 11 + c] = np.float32((rng.uniform(0.25, 0.75) - 0.5) / 0.28209479177387814)
        active = (sh_degree + 1) ** 2
        for k in range(1, active):
            for c in range(3):
                rows[i, 11 + k * 3 + c] = np.float32(rng.normal() * 0.03)
    fx = 0.9 * img
    cam = look_at([0, 0, -2.2], [0, 0, 0], fx, fx, img, img, 0.1, 50.0)
    gt = np.array([rng.uniform(0.0, 1.0) for _ in range(img * img * 3)], np.float64).astype(np.float32)
    return rows, cam, gt.reshape(img, img, 3)


def ref_plan_densify(rows, norm, cnt, dcfg, extent, seed):
    """The reference plan_densify (trainer.hpp:166-213) on a host snapshot: (survivors, children, counts)."""
    rows = np.ascontiguousarray(rows, np.float32)
    n = rows.shape[0]
    norm = np.ascontiguousarray(norm, np.float64)
    cnt = np.ascontiguousarray(cnt, np.int32)
    surv = np.zeros(max(n, 1), np.int32)
    kids = np.zeros((max(2 * n, 1), 59), np.float32)
    counts = np.zeros(5, np.int64)
    d = np.asarray(dcfg, np.float64)
    ref().ref_plan_densify(n, _p(rows), _p(norm), _p(cnt), _p(d), float(extent), int(seed), _p(surv), _p(kids),
                           _p(counts))
    return surv[: counts[0]], kids[: counts[1]], counts


def ref_compute_split_points(geo, cams, mem_limit):
    """compute_split_points (splitter.hpp:31-81): per camera (split, column, left, right, evals), used ratios."""
    geo = np.ascontiguousarray(geo, np.float32)
    cams = np.ascontiguousarray(cams, np.float32)
    out = np.zeros((cams.shape[0], 5), np.int32)
    ratio = np.zeros(cams.shape[0], np.float64)
    ref().ref_compute_split_points(_p(geo), geo.shape[0], cams.shape[0], _p(cams), float(mem_limit), _p(out),
                                   _p(ratio))
    return out, ratio


def ref_psnr_over_views(rows, cams, gts, sh_degree=3):
    rows = np.ascontiguousarray(rows, np.float32)
    cams = np.ascontiguousarray(cams, np.float32)
    gts = np.ascontiguousarray(gts, np.float32)
    exact = np.zeros(1, np.int32)
    db = ref().ref_psnr_over_views(rows.shape[0], _p(rows), cams.shape[0], _p(cams), _p(gts), sh_degree, _p(exact))
    return db, bool(exact[0])


def ref_init_gaussians(positions, colors=None, knn=3, min_knn_dist=0.01, init_opacity=0.1):
    pos = np.ascontiguousarray(positions, np.float32)
    col = None if colors is None else np.ascontiguousarray(colors, np.float32)
    m = pos.shape[0]
    rows = np.zeros((m, 59), np.float32)
    st = ref().ref_init_gaussians(_p(pos), _p(col), m, knn, float(min_knn_dist), float(init_opacity), _p(rows))
    assert st == 0, st
    return rows


def ref_load_ply(path):
    """load_ply (ply.cpp:53-199) of the reference: (positions, colors or None) or raises
    RuntimeError('ParseError: ...') with the reference message."""
    m = C.c_int64()
    hc = C.c_int()
    err = C.create_string_buffer(512)
    st = ref().ref_load_ply(str(path).encode(), C.c_int64(-1), None, None, C.byref(m), C.byref(hc), err, 512)
    if st == 4:
        raise RuntimeError("ParseError: " + err.value.decode())
    assert st == 0, st
    pos = np.zeros((max(m.value, 1), 3), np.float32)
    col = np.zeros((max(m.value, 1), 3), np.float32)
    st = ref().ref_load_ply(str(path).encode(), C.c_int64(m.value), _p(pos), _p(col), C.byref(m), C.byref(hc), err, 512)
    assert st == 0, st
    return pos[: m.value], (col[: m.value] if hc.value else None)


def ref_save_ply(path, pos, col=None, binary=True):
    pos = np.ascontiguousarray(pos, np.float32)
    c = None if col is None else np.ascontiguousarray(col, np.float32)
    assert ref().ref_save_ply(str(path).encode(), _p(pos), None if c is None else _p(c), pos.shape[0],
                              1 if binary else 0) == 0
