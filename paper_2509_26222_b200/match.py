"""Feature correspondences over the C-ABI.

Mirrors terralio::match (/root/reference/proj/core/include/terralio/match/
local_map.hpp, scan_matcher.hpp): ``LocalMap`` (sliding window of frames,
per-frame voxel thinning, edge / planar neighbour structures),
``build_correspondences`` (kNN line / plane fits with the reference's gates
and trims) and the feature rows of ``total_cost`` reduced to normal
equations, which add to the manifold rows' (``kinematics.manifold_rows``) in
one LM step. All numerics run on the device.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, fields

import numpy as np

from . import _abi
from ._abi import InvalidArgument, NormalEqC, check
from .kinematics import NormalEq
from .terrain import Context, _col, _is_dev, _mem, _ptr

EDGE, PLANAR, GROUND = 0, 1, 2  # FeatureKind (types.hpp:36)


class MatchConfigC(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "corr_gate", "huber_delta", "plane_fit_tol", "plane_eig_ratio", "edge_eig_ratio",
        "edge_fit_tol", "edge_min_extent", "trim_ratio", "trim_floor", "ground_corr_voxel",
        "ground_corr_radius")]


@dataclass
class MatchConfig:
    """The association fields of SolverConfig (scan_matcher.hpp:15-49)."""
    corr_gate: float = 1.0
    huber_delta: float = 0.1
    plane_fit_tol: float = 0.025
    plane_eig_ratio: float = 5.0
    edge_eig_ratio: float = 3.0
    edge_fit_tol: float = 0.05
    edge_min_extent: float = 0.05
    trim_ratio: float = 5.0
    trim_floor: float = 0.003
    ground_corr_voxel: float = 0.25
    ground_corr_radius: float = 4.0

    def _c(self) -> MatchConfigC:
        return MatchConfigC(*[float(getattr(self, f.name)) for f in fields(self)])


@dataclass
class Correspondences:
    kind: np.ndarray      # 0 edge (line), 1 plane
    feature: np.ndarray   # index into the scan's features
    params: np.ndarray    # (n, 7): edge point xyz + direction xyz; plane normal xyz + offset
    weight: np.ndarray
    label: np.ndarray     # majority neighbour label
    dist: np.ndarray
    fitq: np.ndarray

    def __len__(self) -> int:
        return len(self.kind)


def _soa3(points):
    return _col(points, 0), _col(points, 1), _col(points, 2)


def _u8(a, like):
    if _is_dev(like):
        import torch
        return a.to(torch.uint8).contiguous()
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint8).reshape(-1))


def _i32(a, like):
    if a is None:
        return None
    if _is_dev(like):
        import torch
        return a.to(torch.int32).contiguous()
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def _pose(R, t):
    return (np.ascontiguousarray(np.asarray(R, dtype=np.float64).reshape(9)),
            np.ascontiguousarray(np.asarray(t, dtype=np.float64).reshape(3)))


class LocalMap:
    """local_map.hpp:17-50."""

    def __init__(self, voxel_size: float = 0.1, window: int = 20, ctx: Context | None = None):
        self.ctx = ctx or Context.default()
        h = C.c_void_p()
        check(_abi.load().tlg_map_create(self.ctx.handle, float(voxel_size), int(window),
                                         C.byref(h)))
        self.handle = h

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _abi.load().tlg_map_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def insert(self, points, kinds, labels, R, t) -> None:
        """LocalMap::insert (local_map.cpp:19-45); points (n, 3) sensor frame."""
        px, py, pz = _soa3(points)
        kd = _u8(kinds, px)
        lb = _i32(labels, px)
        if len(kd) != len(px) or (lb is not None and len(lb) != len(px)):
            raise InvalidArgument("points, kinds and labels differ in length")
        Rm, tv = _pose(R, t)
        check(_abi.load().tlg_map_insert(self.handle, _ptr(px), _ptr(py), _ptr(pz), _ptr(kd),
                                         _ptr(lb), len(px), _mem(px), _ptr(Rm), _ptr(tv)))

    def points(self, kind: int):
        lib = _abi.load()
        n = C.c_size_t()
        check(lib.tlg_map_points(self.handle, int(kind), None, None, 0, C.byref(n)))
        xyz = np.empty((n.value, 3))
        lab = np.empty(n.value, dtype=np.int32)
        check(lib.tlg_map_points(self.handle, int(kind), _ptr(xyz), _ptr(lab), n.value,
                                 C.byref(n)))
        return xyz, lab

    def size(self) -> int:
        return len(self.points(EDGE)[0]) + len(self.points(PLANAR)[0])

    def empty(self) -> bool:
        return self.size() == 0


def build_correspondences(points, kinds, R, t, local_map: LocalMap,
                          config: MatchConfig | None = None) -> Correspondences:
    """scan_matcher.cpp:44-183 at the guess pose (R, t)."""
    cfg = (config or MatchConfig())._c()
    px, py, pz = _soa3(points)
    kd = _u8(kinds, px)
    if len(kd) != len(px):
        raise InvalidArgument("points and kinds differ in length")
    Rm, tv = _pose(R, t)
    lib = _abi.load()
    cnt = C.c_size_t()
    check(lib.tlg_build_correspondences(local_map.handle, _ptr(px), _ptr(py), _ptr(pz), _ptr(kd),
                                        len(px), _mem(px), _ptr(Rm), _ptr(tv), C.byref(cfg),
                                        C.byref(cnt)))
    n = cnt.value
    out = Correspondences(np.empty(n, dtype=np.int32), np.empty(n, dtype=np.uint32),
                          np.empty((n, 7)), np.empty(n), np.empty(n, dtype=np.int32),
                          np.empty(n), np.empty(n))
    check(lib.tlg_correspondences_get(local_map.handle, _ptr(out.kind), _ptr(out.feature),
                                      _ptr(out.params), _ptr(out.weight), _ptr(out.label),
                                      _ptr(out.dist), _ptr(out.fitq), n))
    return out


def feature_normal_eq(local_map: LocalMap, R, t) -> NormalEq:
    """Feature rows of total_cost (scan_matcher.cpp:185-216) at (R, t) for the
    map's last correspondences; valid = number of rows."""
    Rm, tv = _pose(R, t)
    ne = NormalEqC()
    check(_abi.load().tlg_feature_normal_eq(local_map.handle, _ptr(Rm), _ptr(tv), C.byref(ne)))
    return NormalEq._from_c(ne)


def combine(*nes: NormalEq) -> NormalEq:
    """Sum of normal equations of stacked row groups (feature + manifold rows
    reduce into one J^T J, scan_matcher.cpp:296-299)."""
    A = sum(n.A for n in nes)
    g = sum(n.g for n in nes)
    return NormalEq(A, g, float(sum(n.cost for n in nes)), int(sum(n.valid for n in nes)))


def lm_step(ne: NormalEq, mu: float, ctx: Context | None = None) -> np.ndarray:
    """scan_matcher.cpp:300-305 on the device: delta = -(A + mu diag(A)^+ +
    1e-3 I)^-1 g (pivoted LDL^T)."""
    ctx = ctx or Context.default()
    c = NormalEqC()
    k = 0
    for i in range(6):
        for j in range(i, 6):
            c.A[k] = float(ne.A[i, j])
            k += 1
    for i in range(6):
        c.g[i] = float(ne.g[i])
    c.cost = float(ne.cost)
    c.valid = float(ne.valid)
    delta = np.empty(6)
    check(_abi.load().tlg_lm_step(ctx.handle, C.byref(c), float(mu), _ptr(delta)))
    return delta
