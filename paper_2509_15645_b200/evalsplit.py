"""Evaluation and view splitting over the device kernels.

    psnr_over_views         trainer.hpp:131-145 (MSE pooled over views, one PSNR; fp64 device sums)
    compute_split_points    splitter.hpp:31-81 (balance-aware 2-way split search, 5 bisection steps,
                            every evaluation two exact device culls)
    balanced_strip_bounds   the same search generalised to N column strips for image-parallel
                            rendering (imgpar.py): whole-tile cuts balancing the visible counts
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

import numpy as np
import torch

from . import gss as G
from ._abi import GssViewport, check, lib


def image_sq_err(a: torch.Tensor, b: torch.Tensor) -> float:
    """sum (double(a) - double(b))^2 over all elements (image_mse numerator, trainer.hpp:113-122)."""
    if a.shape != b.shape:
        raise ValueError("psnr: image shapes differ")
    out = torch.zeros(1, dtype=torch.float64, device=a.device)
    check(lib().gss_image_sq_err(a.data_ptr(), b.data_ptr(), a.numel(), out.data_ptr(),
                                 torch.cuda.current_stream().cuda_stream))
    return float(out.item())


def psnr_over_views(rows: torch.Tensor, cams: Sequence, gts: Sequence[torch.Tensor], sh_degree: int = 3,
                    background=(0.0, 0.0, 0.0)):
    """psnr_over_views (trainer.hpp:131-145): (dB, exact). rows: device n x 59 (a snapshot)."""
    pooled, elems = 0.0, 0
    for cam, gt in zip(cams, gts):
        img = G.render_view(rows, cam, sh_degree, background)
        n = img.numel()
        pooled += (image_sq_err(img, gt) / n if n else 0.0) * float(n)  # image_mse * size, as the reference
        elems += n
    if elems == 0:
        return 0.0, False
    pooled /= float(elems)
    if pooled == 0.0:
        return math.inf, True
    return 10.0 * math.log10(1.0 / pooled), False


@dataclass
class SplitEntry:
    split: bool = False
    column: int = 0
    used_ratio: float = 0.0
    left_count: int = 0
    right_count: int = 0
    search_evals: int = 0


def _count(geo: torch.Tensor, n: int, cam, vp: GssViewport) -> int:
    return int(G.frustum_cull(geo, n, cam, vp).numel())


def compute_split_points(geo: torch.Tensor, n: int, cams: Sequence, mem_limit: float) -> List[SplitEntry]:
    """compute_split_points (splitter.hpp:31-81) with exact device culls: identical table."""
    table = []
    for cam in cams:
        e = SplitEntry()
        full = _count(geo, n, cam, G.viewport_full(cam.width, cam.height))
        e.used_ratio = full / n if n > 0 else 0.0
        table.append(e)
        if e.used_ratio <= mem_limit or cam.width < 2:
            continue

        def pair(c):
            return (_count(geo, n, cam, GssViewport(0.0, float(c), 0.0, float(cam.height))),
                    _count(geo, n, cam, GssViewport(float(c), float(cam.width), 0.0, float(cam.height))))

        lo, hi = 0, cam.width
        c = cam.width // 2
        left, right = pair(c)
        best = (c, left, right, abs(left - right))
        for _ in range(5):  # kSplitSearchSteps
            if left > right:
                hi = c
            else:
                lo = c
            c = (lo + hi) // 2
            left, right = pair(c)
            e.search_evals += 1
            if abs(left - right) < best[3]:
                best = (c, left, right, abs(left - right))
        bc, bl, br, _ = best
        if bc <= 0 or bc >= cam.width:
            bc = cam.width // 2
            bl, br = pair(bc)
        e.split, e.column, e.left_count, e.right_count = True, bc, bl, br
    return table


def balanced_strip_bounds(count_upto: Callable[[int], int], px0: int, pw: int, nstrips: int,
                          align: int = 16) -> List[int]:
    """N column strips over [px0, px0 + pw) with whole-tile cuts: cut k is the tile boundary c at
    which the visible count of [px0, c) first reaches k/N of the total (count_upto(c) is that
    count; monotone in c — the device cull of viewport [px0, c)). For image-parallel rendering the
    count sums every shard's cull (one all-reduce per evaluation)."""
    tiles = -(-pw // align)
    cuts = [px0 + t * align for t in range(tiles)] + [px0 + pw]
    total = count_upto(px0 + pw)
    bounds = [px0]
    lo_t = 0
    for k in range(1, nstrips):
        target = total * k / nstrips
        lo, hi = lo_t, tiles  # smallest tile index t with count_upto(cuts[t]) >= target
        while lo < hi:
            mid = (lo + hi) // 2
            if count_upto(cuts[mid]) >= target:
                hi = mid
            else:
                lo = mid + 1
        lo_t = lo
        bounds.append(cuts[lo])
    bounds.append(px0 + pw)
    return bounds
