"""The per-scan odometry loop of pipeline.cpp:196-300 (run_odometry) on the
device components, for the C2 configuration: constant-velocity
prediction (the reference's use_imu = false branch; IMU preintegration is out
of scope), lm_solve with the feature rows and the wheel manifold rows,
the cost-history insert gate, LocalMap::insert, select_ground_points and the
terrain model's recursive_update with births.

Control flow and the 6-DoF state live on the host (O(1) per scan); all
data-sized work runs on the device.
"""
from __future__ import annotations

import time
from collections import deque
from dataclasses import dataclass, field

import numpy as np

from . import match as M
from . import terrain as T
from .consumers import select_ground_points


@dataclass
class RunConfig:
    """pipeline.hpp:17-45 (the fields this loop uses)."""
    kernel: T.KernelParams = field(default_factory=T.KernelParams)
    mesh_resolution: float = 0.07
    accept_radius: float = 0.12
    accept_count: int = 3
    map_voxel: float = 0.1
    map_window: int = 20
    solver: M.SolverConfig = field(default_factory=M.SolverConfig)
    use_manifold: bool = True
    ground_voxel: float = 0.12
    ground_radius: float = 2.5
    ground_max_points: int = 400


@dataclass
class FrameDiagnostics:
    index: int = 0
    held: bool = False
    inserted: bool = False
    solve: M.SolveReport | None = None
    terrain: T.UpdateReport | None = None
    ms: dict = field(default_factory=dict)


@dataclass
class RunResult:
    trajectory: list = field(default_factory=list)     # (R, t) per scan
    frames: list = field(default_factory=list)
    terrain: T.TerrainModel | None = None
    local_map: M.LocalMap | None = None


def _arms_at(lever_arms, k):
    if lever_arms is None:
        return None
    if callable(lever_arms):
        return lever_arms(k)
    a = lever_arms if isinstance(lever_arms, (list, tuple)) else np.asarray(lever_arms)
    if isinstance(a, np.ndarray) and a.ndim == 2:
        return a
    return None if a[k] is None else np.asarray(a[k], dtype=np.float64)


def run_odometry(scans, kinds, timestamps, R_first, t_first, roi: T.Rect,
                 lever_arms=None, wheel_radius: float = 0.0,
                 config: RunConfig | None = None) -> RunResult:
    """scans[k]: (n_k, 3) sensor-frame feature points, kinds[k]: FeatureKind
    codes; lever_arms: the (2, 3) wheel-centre offsets in the base frame (the
    leg_model.cpp forward kinematics result) — one array for every frame, a
    per-frame sequence (entries may be None: no joint sample), or a callable
    k -> array | None; None disables the wheel rows."""
    cfg = config or RunConfig()
    kernel = T.KernelParams(cfg.kernel.sigma, cfg.kernel.sigma_eps, cfg.kernel.lambda_,
                            cfg.kernel.cutoff_radius)
    kernel.finalize()
    centers = T.CenterSet(np.zeros((0, 2)), cfg.mesh_resolution, cfg.accept_radius,
                          cfg.accept_count, roi)
    res = RunResult(terrain=T.TerrainModel(kernel, centers),
                    local_map=M.LocalMap(cfg.map_voxel, cfg.map_window))
    R = np.asarray(R_first, dtype=np.float64)
    t = np.asarray(t_first, dtype=np.float64)
    v = np.zeros(3)
    cost_history = deque()
    for k, (P, K) in enumerate(zip(scans, kinds)):
        d = FrameDiagnostics(index=k)
        if k > 0:
            dt = timestamps[k] - timestamps[k - 1]
            Rp, tp = R, t + v * dt
            t0 = time.perf_counter()
            arms = _arms_at(lever_arms, k)
            use_m = cfg.use_manifold and arms is not None and res.terrain.num_centers() > 0
            Rs, ts, rep = M.lm_solve(Rp, tp, P, K, res.local_map, cfg.solver,
                                     terrain=res.terrain if use_m else None,
                                     lever_arms=arms if use_m else None,
                                     wheel_radius=wheel_radius)
            d.ms["solve"] = (time.perf_counter() - t0) * 1e3
            d.solve = rep
            if rep.failed:
                Rs, ts = Rp, tp
                d.held = True
            v = (ts - t) / dt
            R, t = Rs, ts
        accept = not d.held
        if k > 0 and accept:
            rows = max(d.solve.correspondence_count, 1)
            per_row = d.solve.final_cost / rows
            if len(cost_history) >= 5:
                med = sorted(cost_history)[len(cost_history) // 2]
                if per_row > max(10.0 * med, 1e-6):
                    accept = False
            if accept:
                cost_history.append(per_row)
                if len(cost_history) > 20:
                    cost_history.popleft()
        d.inserted = accept
        if accept:
            t0 = time.perf_counter()
            res.local_map.insert(P, K, None, R, t)
            t1 = time.perf_counter()
            obs = select_ground_points(P, K, R, t, roi, cfg.ground_radius, cfg.ground_voxel,
                                       cfg.ground_max_points)
            t2 = time.perf_counter()
            if len(obs.z):
                d.terrain = res.terrain.recursive_update(obs)
            t3 = time.perf_counter()
            d.ms.update(map_insert=(t1 - t0) * 1e3, ground=(t2 - t1) * 1e3,
                        terrain_update=(t3 - t2) * 1e3)
        res.trajectory.append((R.copy(), t.copy()))
        res.frames.append(d)
    return res
