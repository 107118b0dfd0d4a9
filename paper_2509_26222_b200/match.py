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
from .terrain import Context, _CtxBound, _col, _is_dev, _mem, _ptr, torch

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


class LocalMap(_CtxBound):
    """local_map.hpp:17-50."""

    def __init__(self, voxel_size: float = 0.1, window: int = 20, ctx: Context | None = None):
        self.ctx = ctx or Context.default()
        h = C.c_void_p()
        check(_abi.load().tlg_map_create(self.ctx.handle, float(voxel_size), int(window),
                                         C.byref(h)))
        self.handle = h

    def __del__(self):
        try:
            if self._h:
                _abi.load().tlg_map_destroy(self._h)
                self._h = None
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


def associate(points, kinds, R, t, local_map: LocalMap, config: MatchConfig | None = None) -> int:
    """scan_matcher.cpp:44-183 at the guess pose (R, t), keeping the
    correspondences on the device (feature_normal_eq reads them); returns
    their count. `points` may be (n, 3) numpy or a tuple of three contiguous
    CUDA tensors (x, y, z) that stay resident across calls."""
    cfg = (config or MatchConfig())._c()
    px, py, pz = points if isinstance(points, (tuple, list)) else _soa3(points)
    kd = _u8(kinds, px)
    if len(kd) != len(px):
        raise InvalidArgument("points and kinds differ in length")
    Rm, tv = _pose(R, t)
    cnt = C.c_size_t()
    check(_abi.load().tlg_build_correspondences(local_map.handle, _ptr(px), _ptr(py), _ptr(pz),
                                                _ptr(kd), len(px), _mem(px), _ptr(Rm), _ptr(tv),
                                                C.byref(cfg), C.byref(cnt)))
    return cnt.value


def build_correspondences(points, kinds, R, t, local_map: LocalMap,
                          config: MatchConfig | None = None) -> Correspondences:
    """scan_matcher.cpp:44-183 at the guess pose (R, t)."""
    lib = _abi.load()
    n = associate(points, kinds, R, t, local_map, config)
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


# ---------------------------------------------------------------------------
# lm_solve (scan_matcher.cpp:257-358). The LM control flow and the SO(3)
# retraction of the 6-DoF state (so3.cpp:16-58) are O(1) host work per step;
# every data-sized computation — association, feature rows, manifold rows,
# their normal equations, the damped solve and the degeneracy probe — runs on
# the device.
@dataclass
class SolverConfig(MatchConfig):
    lambda_manifold: float = 1.0
    lm_init_damping: float = 1e-4
    lm_max_iters: int = 10
    lm_max_inner: int = 8
    lm_max_rejects: int = 12
    tol_dcost: float = 1e-10
    tol_dstate: float = 1e-10
    min_correspondences: int = 10
    manifold_huber_delta: float = 0.05
    degeneracy_eig_min: float = 10.0

    def _c(self) -> MatchConfigC:
        return MatchConfigC(*[float(getattr(self, f.name)) for f in fields(MatchConfig)])


@dataclass
class SolveReport:
    converged: bool = False
    failed: bool = False
    degenerate: bool = False
    outer_iterations: int = 0
    accepted_steps: int = 0
    final_cost: float = 0.0
    correspondence_count: int = 0
    cost_trace: list = None
    smallest_feature_eigenvalue: float = 0.0


def _hat(v):
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def so3_exp(w) -> np.ndarray:
    """so3.cpp:16-27 (Rodrigues, second-order Taylor below theta^2 = 1e-16)."""
    w = np.asarray(w, dtype=np.float64)
    th2 = float(w @ w)
    W = _hat(w)
    if th2 < 1e-16:
        return np.eye(3) + W + 0.5 * (W @ W)
    th = np.sqrt(th2)
    return np.eye(3) + (np.sin(th) / th) * W + ((1.0 - np.cos(th)) / th2) * (W @ W)


def _reorthonormalize(R, tol=1e-9):
    """so3.cpp:47-58."""
    if np.abs(R.T @ R - np.eye(3)).max() <= tol:
        return R
    U, _, Vt = np.linalg.svd(R)
    F = U @ Vt
    if np.linalg.det(F) < 0:
        F = U @ np.diag([1.0, 1.0, -1.0]) @ Vt
    return F


def _retract(R, t, d):
    """scan_matcher.cpp:35-41: R exp(hat(d_theta)), t + d_t."""
    return _reorthonormalize(R @ so3_exp(d[:3])), t + d[3:]


def _ne29(ne: NormalEq) -> NormalEqC:
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
    return c


def lm_solve(R0, t0, points, kinds, local_map: LocalMap, config: SolverConfig | None = None,
             terrain=None, lever_arms=None, wheel_radius: float = 0.0,
             ctx: Context | None = None):
    """Levenberg-Marquardt pose refinement with re-association every outer
    iteration (scan_matcher.cpp:257-358). With a terrain model and lever arms
    (n, 3) the manifold soft-constraint rows join the normal equations.
    Returns (R, t, SolveReport)."""
    from .kinematics import manifold_rows
    cfg = config or SolverConfig()
    ctx = ctx or Context.default()
    lib = _abi.load()
    rep = SolveReport(cost_trace=[])
    R, t = np.asarray(R0, dtype=np.float64), np.asarray(t0, dtype=np.float64)
    use_manifold = terrain is not None and lever_arms is not None and cfg.lambda_manifold > 0.0

    def total_cost(Rc, tc):
        ne = feature_normal_eq(local_map, Rc, tc)
        feat = ne
        if use_manifold:
            _, nm = manifold_rows(terrain, Rc, tc, lever_arms, wheel_radius, cfg.lambda_manifold,
                                  cfg.manifold_huber_delta, want=())
            ne = combine(ne, nm)
        if ne.valid == 0:
            raise _abi.TerralioError("nothing to optimize")
        return ne, feat

    # the scan stays resident on the device across the re-associations
    scan_pts, scan_kinds = points, kinds
    on_dev = _is_dev(points) or (isinstance(points, (tuple, list)) and _is_dev(points[0]))
    if torch is not None and torch.cuda.is_available() and not on_dev:
        dev = f"cuda:{ctx.device}"
        P = np.asarray(points, dtype=np.float64).reshape(-1, 3)
        scan_pts = tuple(torch.from_numpy(np.ascontiguousarray(P[:, j])).to(dev)
                         for j in range(3))
        scan_kinds = torch.from_numpy(
            np.ascontiguousarray(np.asarray(kinds, dtype=np.uint8))).to(dev)
    mu = cfg.lm_init_damping
    rejects = 0
    for _ in range(cfg.lm_max_iters):
        rep.outer_iterations += 1
        ncorr = associate(scan_pts, scan_kinds, R, t, local_map, cfg)
        rep.correspondence_count = ncorr
        if ncorr < cfg.min_correspondences:
            rep.degenerate = True
            break
        ne, feat = total_cost(R, t)
        rep.cost_trace.append(ne.cost)
        rep.final_cost = ne.cost
        lam = C.c_double()
        check(lib.tlg_ne_min_eigenvalue(ctx.handle, C.byref(_ne29(feat)), C.byref(lam)))
        rep.smallest_feature_eigenvalue = lam.value
        if lam.value < cfg.degeneracy_eig_min:
            rep.degenerate = True
        improved = local_converged = False
        moved = 0.0
        for _ in range(cfg.lm_max_inner):
            delta = np.empty(6)
            st = lib.tlg_lm_step(ctx.handle, C.byref(_ne29(ne)), float(mu), _ptr(delta))
            if st != _abi.TLG_OK:
                rep.failed = True
                return np.asarray(R0, dtype=np.float64), np.asarray(t0, dtype=np.float64), rep
            dn = float(np.linalg.norm(delta))
            if dn < cfg.tol_dstate:
                local_converged = True
                break
            Rc, tc = _retract(R, t, delta)
            ne_c, _ = total_cost(Rc, tc)
            if ne_c.cost < ne.cost:
                dcost = ne.cost - ne_c.cost
                R, t, ne = Rc, tc, ne_c
                rep.cost_trace.append(ne.cost)
                rep.final_cost = ne.cost
                mu = max(mu * 0.1, 1e-12)
                rep.accepted_steps += 1
                improved = True
                rejects = 0
                moved += dn
                if dcost < cfg.tol_dcost or dn < cfg.tol_dstate:
                    local_converged = True
                    break
            else:
                mu *= 10.0
                rejects += 1
                if rejects > cfg.lm_max_rejects:
                    if rep.accepted_steps == 0:
                        rep.failed = True
                        return (np.asarray(R0, dtype=np.float64), np.asarray(t0, dtype=np.float64),
                                rep)
                    local_converged = True
                    break
        if local_converged and moved < 1e-9:
            rep.converged = True
            break
        if not improved and not local_converged and rep.accepted_steps > 0:
            rep.converged = True
            break
        if rep.degenerate and not improved:
            break
    return R, t, rep
