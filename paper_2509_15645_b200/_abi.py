"""ctypes binding of include/gss_b200.h (libgss_b200.so, built in-tree by build.py).

The library is the product: loading fails loudly when it is missing, and there is no CPU
fallback — on a machine without a GPU every compute entry point returns GSS_ERR_CUDA.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# GSS_LIB overrides the library path (kernel-variant experiments built by tools/build_variant.py).
LIB_PATH = Path(os.environ.get("GSS_LIB") or Path(__file__).resolve().parent / "libgss_b200.so")

GSS_OK, GSS_ERR_CUDA, GSS_ERR_INVALID, GSS_ERR_INVARIANT, GSS_ERR_PARSE = 0, 1, 2, 3, 4


class GssCamera(C.Structure):
    """Camera<float> (scene.hpp:77-84), 80 bytes."""

    _fields_ = [
        ("rot", C.c_float * 9),
        ("trans", C.c_float * 3),
        ("fx", C.c_float),
        ("fy", C.c_float),
        ("cx", C.c_float),
        ("cy", C.c_float),
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("near_plane", C.c_float),
        ("far_plane", C.c_float),
    ]


class GssViewport(C.Structure):
    _fields_ = [("x0", C.c_float), ("x1", C.c_float), ("y0", C.c_float), ("y1", C.c_float)]


class GssGroup(C.Structure):
    _fields_ = [
        ("col0", C.c_int32),
        ("dim", C.c_int32),
        ("lr", C.c_double),
        ("beta1", C.c_double),
        ("beta2", C.c_double),
        ("eps", C.c_double),
    ]


class GssArena(C.Structure):
    _fields_ = [
        ("w", C.c_void_p),
        ("m", C.c_void_p),
        ("v", C.c_void_p),
        ("counter", C.c_void_p),
        ("n", C.c_int64),
        ("dim", C.c_int32),
        ("defer_max", C.c_int32),
        ("step", C.c_int64),
        ("ngroups", C.c_int32),
        ("groups", GssGroup * 8),
        ("row_stride", C.c_int64),
    ]


class GssSparseGrads(C.Structure):
    _fields_ = [
        ("ids", C.c_void_p),
        ("count", C.c_int64),
        ("count_dev", C.c_void_p),
        ("rows", C.c_void_p),
        ("stride", C.c_int64),
        ("col0", C.c_int32),
    ]


class GssRenderScene(C.Structure):
    _fields_ = [
        ("ids", C.c_void_p),
        ("count", C.c_int64),
        ("count_dev", C.c_void_p),
        ("geo", C.c_void_p),
        ("geo_stride", C.c_int64),
        ("nongeo", C.c_void_p),
        ("nongeo_stride", C.c_int64),
        ("nongeo_compact", C.c_int32),
        ("slot_map", C.c_void_p),
        ("sh_degree", C.c_int32),
        ("background", C.c_float * 3),
        ("low_pass", C.c_float),
    ]


class GssEngineConfig(C.Structure):
    _fields_ = [
        ("lr_mean", C.c_double),
        ("lr_scale", C.c_double),
        ("lr_quat", C.c_double),
        ("lr_opacity", C.c_double),
        ("lr_sh", C.c_double),
        ("sh_rest_divisor", C.c_double),
        ("beta1", C.c_double),
        ("beta2", C.c_double),
        ("eps", C.c_double),
        ("scene_extent", C.c_double),
        ("defer_max", C.c_int32),
        ("geo_defer_max", C.c_int32),
        ("pipelined", C.c_int32),
        ("sh_degree", C.c_int32),
        ("sh_warmup_step", C.c_int32),
        ("background", C.c_float * 3),
        ("low_pass", C.c_float),
        ("nongeo_on_host", C.c_int32),
        ("chunk_bytes", C.c_int64),
    ]


class GssDensifyConfig(C.Structure):
    _fields_ = [("grad_threshold", C.c_double), ("percent_dense", C.c_double), ("opacity_prune", C.c_double),
                ("split_scale_divisor", C.c_double)]


P, I64, I32, F32, F64, SZ = C.c_void_p, C.c_int64, C.c_int32, C.c_float, C.c_double, C.c_size_t

# name -> (restype, argtypes); the exported symbol set of include/gss_b200.h.
SIGNATURES = {
    "gss_last_error": (C.c_char_p, []),
    "gss_abi_version": (I32, []),
    "gss_device_count": (I32, []),
    "gss_launch_count": (I64, []),
    "gss_expf_device": (C.c_int, [P, P, I64, P]),
    "gss_cull_workspace_bytes": (SZ, [I64]),
    "gss_cull": (C.c_int, [P, I64, I64, C.POINTER(GssCamera), C.POINTER(GssViewport), F32, P, P, P, P, SZ, P]),
    "gss_build_group_luts": (C.c_int, [F64, F64, F64, F64, I64, I32, P, P, P, P, P, P]),
    "gss_adam_step_dense": (C.c_int, [C.POINTER(GssArena), P, P]),
    "gss_deferred_update": (C.c_int, [C.POINTER(GssArena), C.POINTER(GssSparseGrads), P, P, P]),
    "gss_restore_view": (C.c_int, [C.POINTER(GssArena), P, I64, P, C.POINTER(GssSparseGrads), P, P]),
    "gss_flush_deferred": (C.c_int, [C.POINTER(GssArena), P]),
    "gss_arena_check": (C.c_int, [C.POINTER(GssArena), P]),
    "gss_arena_release": (C.c_int, [C.POINTER(GssArena)]),
    "gss_cull_workspace_release": (None, [P]),
    "gss_render_ctx_create": (P, []),
    "gss_render_ctx_destroy": (None, [P]),
    "gss_rasterize_forward": (C.c_int, [P, C.POINTER(GssRenderScene), C.POINTER(GssCamera),
                                        C.POINTER(GssViewport), P, P, I64, P, P, P, P, P, P]),
    "gss_loss_l1": (C.c_int, [P, P, I64, I64, P, P, P]),
    "gss_rasterize_backward": (C.c_int, [P, P, P, I64, P, I64, P, P]),
    "gss_image_sq_err": (C.c_int, [P, P, I64, P, P]),
    "gss_project": (C.c_int, [C.POINTER(GssRenderScene), C.POINTER(GssCamera), C.POINTER(GssViewport), P, P]),
    "gss_route_strips": (C.c_int, [P, I64, P, I32, P, P, P]),
    "gss_gather_records": (C.c_int, [P, P, I64, P, P]),
    "gss_scatter_add_rows": (C.c_int, [P, P, I64, I32, P, P]),
    "gss_rasterize_records_forward": (C.c_int, [P, P, I64, C.POINTER(GssCamera), C.POINTER(GssViewport), P, P, P,
                                                I64, P, P, P, P, P, P, P]),
    "gss_rasterize_records_backward": (C.c_int, [P, P, P, P]),
    "gss_chain_backward": (C.c_int, [C.POINTER(GssRenderScene), C.POINTER(GssCamera), P, P, P, I64, P, I64, P, P]),
    "gss_engine_config_default": (None, [C.POINTER(GssEngineConfig)]),
    "gss_plan_densify": (C.c_int, [P, I64, P, P, C.POINTER(GssDensifyConfig), F64, C.c_uint64, P, P, P, P]),
    "gss_engine_densify": (C.c_int, [P, C.POINTER(GssDensifyConfig), F64, C.c_uint64, P]),
    "gss_engine_create": (P, [I64, P, I32, P, P, C.POINTER(GssEngineConfig)]),
    "gss_engine_destroy": (None, [P]),
    "gss_engine_run": (C.c_int, [P, I32, P, P]),
    "gss_engine_step": (C.c_int, [P, C.POINTER(GssCamera), P, P, P]),
    "gss_engine_step_async": (C.c_int, [P, C.POINTER(GssCamera), P, P, P]),
    "gss_engine_drain": (C.c_int, [P]),
    "gss_engine_set_splits": (C.c_int, [P, C.c_int32, P, P]),
    "gss_set_host_chunk_bytes": (C.c_int, [C.c_int64]),
    "gss_engine_snapshot": (C.c_int, [P, P]),
    "gss_engine_state": (C.c_int, [P, P, P, P, P, P, P]),
    "gss_engine_accum": (C.c_int, [P, P, P]),
    "gss_engine_count": (I64, [P]),
    "gss_engine_stage_ms": (C.c_int, [P, P]),
    "gss_engine_launches": (I64, [P]),
    "gss_synth_scene": (C.c_int, [C.c_uint64, I64, I32, I32, I32, I32, P, P, P]),
    "gss_init_gaussians": (C.c_int, [P, P, I32, I32, F64, F64, P]),
    "gss_look_at_camera": (C.c_int, [P, P, F32, F32, I32, I32, F32, F32, C.POINTER(GssCamera)]),
    "gss_raster_stats": (C.c_int, [P, I32]),
    "gss_arena_access": (C.c_int, [C.POINTER(GssArena), P]),
    "gss_engine_kernel_timing": (C.c_int, [P, I32]),
    "gss_engine_timeline_enable": (C.c_int, [P, I32]),
    "gss_engine_timeline": (I64, [P, P, I64]),
    "gss_engine_stage_delays": (C.c_int, [P, P, I32]),
    "gss_engine_kernel_times": (C.c_int, [P, P, P, P]),
    "gss_engine_render_times": (C.c_int, [P, P, P, P]),
    "gss_raster_stats_enabled": (I32, []),
    "gss_ply_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "gss_ply_read": (C.c_int, [P, P, P, P]),
    "gss_ply_close": (None, [P]),
    "gss_save_ply": (C.c_int, [C.c_char_p, P, P, I64, I32]),
}

_lib = None


def lib() -> C.CDLL:
    """The loaded libgss_b200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2509_15645_b200.build` "
                "(there is no CPU fallback for the hot path)")
        l = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(l, name)
            f.restype = res
            f.argtypes = args
        _lib = l
    return _lib


class GssError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class ConfigError(GssError):
    """Reference ConfigError / std::invalid_argument (status 2)."""


class InvariantViolation(GssError):
    """Reference InvariantViolation (status 3)."""


class ParseError(GssError):
    """Reference ParseError (status 4; PLY ingestion)."""


def check(status: int) -> None:
    if status == GSS_OK:
        return
    msg = lib().gss_last_error().decode(errors="replace")
    if status == GSS_ERR_INVALID:
        raise ConfigError(status, msg)
    if status == GSS_ERR_INVARIANT:
        raise InvariantViolation(status, msg)
    if status == GSS_ERR_PARSE:
        raise ParseError(status, msg)
    raise GssError(status, msg)
