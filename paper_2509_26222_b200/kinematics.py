"""Wheel/ground manifold soft constraint over the C-ABI.

Mirrors terralio::kin (contact.hpp:15-24, leg_model.hpp:32-60) and the
manifold block of match::total_cost (scan_matcher.cpp:221-248). The batched
entry point `manifold_rows` is the B200 hot path: one kernel computes every
row's residual and 1x6 Jacobian and reduces J^T J, J^T r and the cost in the
same pass (tlg_manifold_rows).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from ._abi import InvalidArgument, NormalEqC, check
from .terrain import TerrainModel, _empty_like, _is_dev, _mem, _ptr

try:
    import torch
except Exception:  # pragma: no cover
    torch = None


@dataclass
class NormalEq:
    """A = J^T J (6x6), g = J^T r, cost = |r|^2 (scan_matcher.cpp:296-299,253)."""
    A: np.ndarray
    g: np.ndarray
    cost: float
    valid: int

    @staticmethod
    def _from_c(c: NormalEqC) -> "NormalEq":
        v = np.frombuffer(c, dtype=np.float64)  # A[21] (upper, row-major), g[6], cost, valid
        A = np.empty((6, 6))
        A[_IU] = v[:21]
        A[_IU[1], _IU[0]] = v[:21]
        return NormalEq(A, v[21:27].copy(), float(v[27]), int(round(v[28])))


_IU = np.triu_indices(6)


def manifold_rows(terrain: TerrainModel, R, t, h, wheel_radius: float = 0.0,
                  lambda_M: float = 1.0, huber_delta: float = 0.05,
                  want=("r", "J", "valid"), out: dict | None = None):
    """Rows r_i = sqrt(lambda_M) w_i (xi_z - wheel_radius - f(xi_xy)),
    xi = R h_i + t, with their Jacobians (column-major n x 6 like
    CostEval::jacobian) and the fused normal equations.

    h: (n, 3) lever arms or an SoA tuple (hx, hy, hz) of contiguous float64
    arrays (numpy = host, torch CUDA = device). Returns
    (rows: dict[str, array], NormalEq).
    """
    Rm = np.ascontiguousarray(np.asarray(R, dtype=np.float64).reshape(9))
    tv = np.ascontiguousarray(np.asarray(t, dtype=np.float64).reshape(3))
    if isinstance(h, (tuple, list)):  # SoA (hx, hy, hz), used as-is (no copies)
        hx, hy, hz = h
    elif _is_dev(h):
        hx, hy, hz = (h[:, j].to(torch.float64).contiguous() for j in range(3))
    else:
        ha = np.asarray(h, dtype=np.float64).reshape(-1, 3)
        hx, hy, hz = (np.ascontiguousarray(ha[:, j]) for j in range(3))
    n = len(hx)
    rows = dict(out or {})
    for key, dt, size in (("r", np.float64, n), ("J", np.float64, 6 * n), ("valid", np.uint8, n),
                          ("raw", np.float64, n)):
        if key in want and key not in rows:
            rows[key] = _empty_like(hx, size, dt)
    # rows go where the caller's buffers live (host lever arms may feed
    # device rows: the streamed H2D path of tlg_manifold_rows)
    outs = [v for v in rows.values() if v is not None]
    out_mem = _mem(outs[0]) if outs else _mem(hx)
    if any(_mem(v) != out_mem for v in outs):
        raise InvalidArgument("row buffers must all be host or all be device memory")
    ne = NormalEqC()
    check(_abi.load().tlg_manifold_rows(
        terrain.handle, _ptr(Rm), _ptr(tv), _ptr(hx), _ptr(hy), _ptr(hz), n, _mem(hx),
        float(wheel_radius), float(lambda_M), float(huber_delta), _ptr(rows.get("r")),
        _ptr(rows.get("J")), _ptr(rows.get("valid")), _ptr(rows.get("raw")), out_mem,
        C.byref(ne)))
    return rows, NormalEq._from_c(ne)


class Scan:
    """A scan's lever arms binned on the device by world cell under pose
    (R0, t0) (tlg_scan_create). manifold_rows() rows come out in scan order;
    permutation()[k] is the input index of row k."""

    def __init__(self, terrain: TerrainModel, R0, t0, h):
        Rm = np.ascontiguousarray(np.asarray(R0, dtype=np.float64).reshape(9))
        tv = np.ascontiguousarray(np.asarray(t0, dtype=np.float64).reshape(3))
        if isinstance(h, (tuple, list)):
            hx, hy, hz = h
        elif _is_dev(h):
            hx, hy, hz = (h[:, j].to(torch.float64).contiguous() for j in range(3))
        else:
            ha = np.asarray(h, dtype=np.float64).reshape(-1, 3)
            hx, hy, hz = (np.ascontiguousarray(ha[:, j]) for j in range(3))
        self.terrain = terrain
        self.n = len(hx)
        self._dev = _is_dev(hx)
        self._ref = hx
        self._pose = np.zeros(12)  # R (9) then t (3), reused by every evaluation
        self._pose_p = self._pose.ctypes.data
        self._ne = NormalEqC()
        self._ne_ref = C.byref(self._ne)
        hdl = C.c_void_p()
        check(_abi.load().tlg_scan_create(terrain.handle, _ptr(Rm), _ptr(tv), _ptr(hx), _ptr(hy),
                                          _ptr(hz), self.n, _mem(hx), C.byref(hdl)))
        self.handle = hdl

    def bin_ms(self) -> float:
        n, ms = C.c_size_t(), C.c_double()
        check(_abi.load().tlg_scan_info(self.handle, C.byref(n), C.byref(ms)))
        return ms.value

    def permutation(self) -> np.ndarray:
        out = np.empty(self.n, dtype=np.uint32)
        check(_abi.load().tlg_scan_permutation(self.handle, _ptr(out), _abi.TLG_HOST))
        return out

    def manifold_rows(self, R, t, wheel_radius=0.0, lambda_M=1.0, huber_delta=0.05,
                      want=("r", "J", "valid"), out: dict | None = None, device_out=None):
        # called once per LM cost evaluation: a lean path (pose into a
        # reused buffer, the caller's row buffers as-is)
        pose = self._pose
        pose[:9] = np.asarray(R, dtype=np.float64).reshape(9)
        pose[9:] = np.asarray(t, dtype=np.float64).reshape(3)
        dev = self._dev if device_out is None else device_out
        n = self.n
        if out is not None and all(k in out for k in want):
            rows = out
        else:
            ref = self._ref if dev else np.empty(0)
            rows = dict(out or {})
            for key, dt, size in (("r", np.float64, n), ("J", np.float64, 6 * n),
                                  ("valid", np.uint8, n), ("raw", np.float64, n)):
                if key in want and key not in rows:
                    rows[key] = _empty_like(ref, size, dt)
        mem = _abi.TLG_DEVICE if dev else _abi.TLG_HOST
        ne = self._ne
        get = rows.get
        check(_abi.load().tlg_scan_manifold_rows(
            self.terrain.handle, self.handle, self._pose_p, self._pose_p + 72, float(wheel_radius),
            float(lambda_M), float(huber_delta), _ptr(get("r")), _ptr(get("J")),
            _ptr(get("valid")), _ptr(get("raw")), mem, self._ne_ref))
        return rows, NormalEq._from_c(ne)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                _abi.load().tlg_scan_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Leg model (leg_model.hpp:14-60): host-side forward kinematics that produces
# the two wheel lever arms; scalar bookkeeping, not the data path.
@dataclass
class Link:
    name: str = ""
    parent: str = ""
    offset: tuple = (0.0, 0.0, 0.0)
    axis: tuple = (0.0, 1.0, 0.0)
    revolute: bool = True


@dataclass
class LegChain:
    links: list = field(default_factory=list)

    def joint_count(self) -> int:
        return sum(1 for l in self.links if l.revolute)


@dataclass
class LegModel:
    left: LegChain = field(default_factory=LegChain)
    right: LegChain = field(default_factory=LegChain)
    wheel_radius: float = 0.1

    def joint_count(self) -> int:
        return self.left.joint_count() + self.right.joint_count()

    def chain(self, side: str) -> LegChain:
        return self.left if side == "left" else self.right

    def joint_offset(self, side: str) -> int:
        return 0 if side == "left" else self.left.joint_count()


def _axis_angle(axis, angle):
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + math.sin(angle) * K + (1 - math.cos(angle)) * (K @ K)


def chain_end_position(chain: LegChain, q) -> np.ndarray:
    """leg_model.cpp:10-21: translate by each offset, then rotate revolute links."""
    if len(q) < chain.joint_count():
        raise _abi.InvalidArgument("too few joint angles for chain")
    Rm, p, qi = np.eye(3), np.zeros(3), 0
    for link in chain.links:
        p = p + Rm @ np.asarray(link.offset, dtype=np.float64)
        if link.revolute:
            Rm = Rm @ _axis_angle(link.axis, q[qi])
            qi += 1
    return p


def default_robot() -> LegModel:
    """sim::default_robot (scene.cpp:12-28)."""
    def chain(ys):
        return LegChain([Link("hip", "base", (0.0, ys * 0.12, -0.08), (0, 1, 0), True),
                         Link("knee", "hip", (0.0, 0.0, -0.24), (0, 1, 0), True),
                         Link("wheel", "knee", (0.0, 0.0, -0.24), (0, 1, 0), False)])
    return LegModel(chain(1.0), chain(-1.0), 0.08)


def lever_arm(leg: LegModel, joints, side: str) -> np.ndarray:
    off = leg.joint_offset(side)
    ch = leg.chain(side)
    if len(joints) < leg.joint_count():
        raise _abi.InvalidArgument("joint config does not match leg model")
    return chain_end_position(ch, list(joints)[off: off + ch.joint_count()])


@dataclass
class ManifoldResidual:
    value: float = 0.0
    valid: bool = False
    wheel_center: np.ndarray = field(default_factory=lambda: np.zeros(3))


def manifold_residual(R, t, joints, leg: LegModel, side: str,
                      terrain: TerrainModel) -> ManifoldResidual:
    """contact.cpp:7-19 (wheel row through the batched kernel, n = 1)."""
    h = lever_arm(leg, joints, side)
    rows, _ = manifold_rows(terrain, R, t, h.reshape(1, 3), leg.wheel_radius, 1.0, 0.0,
                            want=("raw", "valid"))
    wc = np.asarray(R, dtype=np.float64).reshape(3, 3) @ h + np.asarray(t, dtype=np.float64)
    ok = bool(rows["valid"][0])
    return ManifoldResidual(float(rows["raw"][0]) if ok else 0.0, ok, wc)


def manifold_jacobian(R, t, joints, leg: LegModel, side: str, terrain: TerrainModel) -> np.ndarray:
    """contact.cpp:21-39: d r / d [dtheta, dt] (right perturbation)."""
    h = lever_arm(leg, joints, side)
    rows, _ = manifold_rows(terrain, R, t, h.reshape(1, 3), leg.wheel_radius, 1.0, 0.0,
                            want=("J", "valid"))
    J = np.asarray(rows["J"]).reshape(6)
    if not rows["valid"][0]:
        # unsupported query: the reference's predict_gradient is 0 -> [0,0,1]*dxi
        Rm = np.asarray(R, dtype=np.float64).reshape(3, 3)
        dr = np.array([0.0, 0.0, 1.0])
        u = Rm.T @ dr
        return np.concatenate([np.cross(h, u), dr])
    return J
