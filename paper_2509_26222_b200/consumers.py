"""Batch-predict consumers on either side of the update,
over the C-ABI:

* ``select_ground_points`` — pipeline.cpp:150-170 (anonymous-namespace helper
  of the pipeline): ground-labelled scan points to the world frame, ROI and
  radius filter, first point per xy voxel in scan order, capped;
* ``terrain_error_histogram`` / ``Histogram`` — metrics.hpp:42-51,
  metrics.cpp:184-232;
* ``export_csv`` — TerrainModel::export_csv (terrain_model.cpp:255-267): the
  grid walk is the reference's (x outer, y inner, ``+= grid_step``
  accumulation, ``<= max + 1e-12``), the heights come from one batched device
  evaluation, the text is ostream's default ``%g`` formatting.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import InvalidArgument, TerralioError, check
from .terrain import (Context, Rect, TerrainModel, TerrainObservation, _col, _is_dev, _mem,
                      _ptr, _same_space, _vec)

GROUND = 2  # FeatureKind::Ground (types.hpp:36)


def select_ground_points(points, kinds, R, t, roi: Rect, ground_radius: float = 2.5,
                         ground_voxel: float = 0.12, ground_max_points: int = 400,
                         ctx: Context | None = None) -> TerrainObservation:
    """points: (n, 3) sensor-frame points (numpy or torch CUDA), kinds: (n,)
    FeatureKind codes (uint8). Returns the kept world-frame ground points as
    a TerrainObservation (same memory space as the input)."""
    ctx = ctx or Context.default()
    px, py, pz = _col(points, 0), _col(points, 1), _col(points, 2)
    if _is_dev(points):
        import torch
        kd = kinds.to(torch.uint8).contiguous()
    else:
        kd = np.ascontiguousarray(np.asarray(kinds, dtype=np.uint8).reshape(-1))
    _same_space(px, kd)
    n = len(px)
    if len(kd) != n:
        raise InvalidArgument("points and kinds differ in length")
    Rm = np.ascontiguousarray(np.asarray(R, dtype=np.float64).reshape(9))
    tv = np.ascontiguousarray(np.asarray(t, dtype=np.float64).reshape(3))
    lo = np.array(roi.min, dtype=np.float64)
    hi = np.array(roi.max, dtype=np.float64)
    cap = max(int(ground_max_points), 1)
    if _is_dev(px):
        import torch
        ox, oy, oz = (torch.empty(cap, dtype=torch.float64, device=px.device) for _ in range(3))
    else:
        ox, oy, oz = np.empty(cap), np.empty(cap), np.empty(cap)
    kept = C.c_size_t()
    check(_abi.load().tlg_select_ground_points(
        ctx.handle, _ptr(px), _ptr(py), _ptr(pz), _ptr(kd), n, _mem(px), _ptr(Rm), _ptr(tv),
        _ptr(lo), _ptr(hi), float(ground_radius), float(ground_voxel), int(ground_max_points),
        _ptr(ox), _ptr(oy), _ptr(oz), _mem(px), C.byref(kept)))
    k = kept.value
    if _is_dev(px):
        import torch
        return TerrainObservation(torch.stack([ox[:k], oy[:k]], 1), oz[:k].clone())
    return TerrainObservation(np.stack([ox[:k], oy[:k]], 1), oz[:k].copy())


# metrics.hpp:42-51
@dataclass
class Histogram:
    edges: np.ndarray = field(default_factory=lambda: np.zeros(0))
    counts: np.ndarray = field(default_factory=lambda: np.zeros(0, dtype=np.uint64))
    trimmed: int = 0
    overflow: int = 0

    def total(self) -> int:
        """metrics.cpp:184-188."""
        return int(self.overflow + int(self.counts.sum()))

    def fraction_below(self, threshold: float) -> float:
        """metrics.cpp:190-197."""
        n = self.total()
        if n == 0:
            return 0.0
        below = sum(int(c) for b, c in enumerate(self.counts)
                    if self.edges[b + 1] <= threshold + 1e-12)
        return below / n


def terrain_error_histogram(model: TerrainModel, xy, z, trim_fraction: float = 0.0,
                            bins: int = 25) -> Histogram:
    """metrics.cpp:199-232: |z - f(xy)| per sample (0.25 m where the model
    has no support), the top floor(trim_fraction n) dropped, binned."""
    x, y = _col(xy, 0), _col(xy, 1)
    zz = _vec(z)
    _same_space(x, zz)
    n = len(x)
    if n == 0 or len(zz) != n:
        raise InvalidArgument("histogram needs matched non-empty samples")
    edges = np.empty(int(bins) + 1)
    counts = np.zeros(max(int(bins), 1), dtype=np.uint64)
    tr, ov = C.c_uint64(), C.c_uint64()
    check(_abi.load().tlg_terrain_error_histogram(
        model.handle, _ptr(x), _ptr(y), _ptr(zz), n, _mem(x), float(trim_fraction), int(bins),
        _ptr(edges), _ptr(counts), C.byref(tr), C.byref(ov)))
    return Histogram(edges, counts[:int(bins)], int(tr.value), int(ov.value))


def export_grid(model: TerrainModel, grid_step: float):
    """The numbers of export_csv: supported grid points (x outer, y inner) and
    their heights, in the reference's order."""
    if not grid_step > 0.0:
        raise InvalidArgument("grid_step must be positive")
    lib = _abi.load()
    cp = _abi.CenterParamsC()
    check(lib.tlg_model_center_params(model.handle, C.byref(cp)))
    roi = Rect((cp.roi_min_x, cp.roi_min_y), (cp.roi_max_x, cp.roi_max_y))
    xs = []
    x = roi.min[0]
    while x <= roi.max[0] + 1e-12:
        xs.append(x)
        x += grid_step
    ys = []
    y = roi.min[1]
    while y <= roi.max[1] + 1e-12:
        ys.append(y)
        y += grid_step
    gx = np.repeat(np.asarray(xs, dtype=np.float64), len(ys))
    gy = np.tile(np.asarray(ys, dtype=np.float64), len(xs))
    z, s, _, _ = model.predict(np.stack([gx, gy], 1), gradient=False)
    keep = s.astype(bool)
    return gx[keep], gy[keep], z[keep]


def export_csv(model: TerrainModel, path: str, grid_step: float) -> None:
    """TerrainModel::export_csv (terrain_model.cpp:255-267)."""
    gx, gy, z = export_grid(model, grid_step)
    try:
        with open(path, "w") as f:
            f.write("x,y,z_pred\n")
            f.writelines(f"{a:g},{b:g},{c:g}\n" for a, b, c in zip(gx, gy, z))
    except OSError as e:
        raise TerralioError(f"cannot open {path}") from e
