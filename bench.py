#!/usr/bin/env python
"""Benchmark of the B200 RBF-terrain hot path (BASELINE.json metric:
"RBF residual+Jacobian evals/s; kernel-matrix update ms/scan (M centers)").

Headline (`value`): manifold soft-constraint rows — residual + 6-DoF
Jacobian per LiDAR point, materialised (r, J column-major, valid) with the
fused J^T J / J^T r / cost reduction — over the C5 workload: 10^7 points per
GPU against a 316 x 316 = 99,856-centre RBF terrain (points/s, whole job).
One step = one LM cost evaluation (tlg_manifold_rows) over all points.

Secondary (`update`): per-scan TerrainModel::recursive_update latency at
M = 4096 centres (C3 staircase), m = 400 (pipeline cap) and m = 20,000.

`--impl reference` times the reference algorithm's CPU path: the plain-C++
oracle restatement (the reference itself cannot be built here)
on the host cores, same metric/config.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RBF residual+Jacobian evals/s (manifold rows + fused 6x6 normal equations)"
UNIT = "points/s"

# C5: ROI [0, 22.05]^2, 316 x 316 lattice, 10^7 points
ROI_C5 = ((0.0, 0.0), (22.05, 22.05))
RES, R_A, COUNT = 0.07, 0.12, 3
POSE_W = (0.02, -0.015, 0.04)           # bench_main.cpp:116
POSE_T = (0.1, -0.05, 0.08)             # bench_main.cpp:117
BYTES_PER_POINT = 24 + 8 + 48 + 1       # h in; r, J[6], valid out


def terrain_c5(x, y, xp):
    """C4/C5 sinusoidal bumps z = 0.05 sin(2 pi x / 1.5) sin(2 pi y / 1.5)."""
    return 0.05 * xp.sin(2 * math.pi * x / 1.5) * xp.sin(2 * math.pi * y / 1.5)


def staircase(x):
    """TerrainSpec::staircase(0.08, 0.5, 10, x0=0.5) (terrain_spec.cpp:72-77)."""
    xr = x - 0.5
    idx = np.floor(xr / 0.5)
    return np.where(xr < 0.0, 0.0, 0.08 * np.minimum(idx, 10.0))


def so3_exp(w):
    """Rodrigues (so3.cpp:16-27), second-order Taylor below theta^2 = 1e-16."""
    w = np.asarray(w, dtype=np.float64)
    th2 = float(w @ w)
    K = np.array([[0, -w[2], w[1]], [w[2], 0, -w[0]], [-w[1], w[0], 0]])
    if th2 < 1e-16:
        return np.eye(3) + K + 0.5 * (K @ K)
    th = math.sqrt(th2)
    return np.eye(3) + math.sin(th) / th * K + (1 - math.cos(th)) / th2 * (K @ K)


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        self.f.flush()
        rows = []
        for line in Path(self.f.name).read_text().splitlines():
            parts = [s.strip() for s in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
def cpu_backend():
    """The CPU side of the bench (cpu_baseline leg / --impl reference only):
    the reference itself compiled from its unchanged sources (oracle/_ref,
    kind "reference") when present, else the plain-C++ restatement ("port")."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc
    ref = orc.reference()
    return (ref, "reference") if ref is not None else (orc, "port")


def cpu_eval_rate(centers_xy, weights, kernel, pts_h, R, t, seconds=10.0, threads=None):
    """The reference's manifold rows (kin::manifold_residual/jacobian with the
    total_cost weighting) on a bounded sample, all host threads."""
    orc, _ = cpu_backend()
    from paper_2509_26222_b200.terrain import CenterSet, Rect
    threads = threads or os.cpu_count() or 1
    cs = CenterSet(centers_xy, RES, R_A, COUNT, Rect(*ROI_C5))
    om = orc.Model(kernel, cs)
    om.set_weights(weights)
    n0 = min(len(pts_h), 20000)
    t0 = time.perf_counter()
    om.manifold_rows(R, t, pts_h[:n0], 0.0, 1.0, 0.05, threads=threads)
    dt = time.perf_counter() - t0
    rate0 = n0 / dt
    n = int(min(len(pts_h), max(n0, rate0 * seconds)))
    t0 = time.perf_counter()
    om.manifold_rows(R, t, pts_h[:n], 0.0, 1.0, 0.05, threads=threads)
    dt = time.perf_counter() - t0
    return n / dt, n, threads, dt, om


def build_c5(device, n_points, seed, torch):
    """C5 model (select_centers on 10^6 support points) + n_points lever arms."""
    from paper_2509_26222_b200 import terrain as T
    g = torch.Generator(device=f"cuda:{device}").manual_seed(seed)
    sup = torch.rand((1_000_000, 2), generator=g, device=f"cuda:{device}", dtype=torch.float64)
    sup *= ROI_C5[1][0]
    zs = terrain_c5(sup[:, 0], sup[:, 1], torch)
    cs = T.select_centers(T.TerrainObservation(sup, zs), T.Rect(*ROI_C5), RES, R_A, COUNT)
    kernel = T.KernelParams()
    kernel.finalize()
    model = T.TerrainModel(kernel, cs)
    c = cs.centers
    # interpolating weights: height * res^2 / (2 pi sigma^2)
    w = terrain_c5(c[:, 0], c[:, 1], np) * RES * RES / (2 * math.pi * kernel.sigma ** 2)
    model.set_weights(w)
    R = so3_exp(POSE_W)
    tv = np.array(POSE_T)
    p = torch.rand((n_points, 2), generator=g, device=f"cuda:{device}", dtype=torch.float64)
    p *= ROI_C5[1][0]
    pz = terrain_c5(p[:, 0], p[:, 1], torch) + 0.01 * torch.randn(
        n_points, generator=g, device=f"cuda:{device}", dtype=torch.float64)
    P = torch.stack([p[:, 0], p[:, 1], pz], 1)
    Rt = torch.from_numpy(R).to(P)
    H = (P - torch.from_numpy(tv).to(P)) @ Rt  # rows: R^T (p - t)
    h = tuple(H[:, j].contiguous() for j in range(3))
    del P, H, p, pz, sup
    return model, kernel, cs, w, R, tv, h


# ---------------------------------------------------------------------------
def run_update_bench(torch, device, steps=5):
    """C3: per-scan recursive_update at M = 4096 (64 x 64 lattice)."""
    from paper_2509_26222_b200 import terrain as T
    roi = T.Rect((0.0, 0.0), (4.41, 4.41))
    kernel = T.KernelParams()
    kernel.finalize()
    model = T.TerrainModel(kernel, T.CenterSet(np.zeros((0, 2)), RES, R_A, COUNT, roi))
    rng = np.random.default_rng(3)

    def scan(m):
        clean = rng.uniform(0.0, 4.41, size=(m, 2))
        noisy = clean + rng.normal(0.0, 0.1, size=(m, 2))
        return T.TerrainObservation(np.ascontiguousarray(noisy), staircase(clean[:, 0]))

    rep0 = model.recursive_update(scan(20000))  # births: all 4096 nodes
    out = {"M": model.num_centers(), "born_first_scan": rep0.born_centers}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for m in (400, 20000):
        scans = [scan(m) for _ in range(steps + 2)]
        for s in scans[:2]:
            model.recursive_update(s)
        times, reps = [], []
        for s in scans[2:]:
            ev0.record()
            rep = model.recursive_update(s)
            ev1.record()
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
            reps.append(rep)
        rep = reps[-1]
        gflop = statistics.median(r.flops for r in reps) / 1e9
        out[f"m{m}"] = {"ms_per_scan": statistics.median(times), "ms_min": min(times),
                        "n_active": rep.active_centers, "active_blocks": rep.active_blocks,
                        "solver": rep.solver, "rejected": rep.rejected,
                        "gflop_per_scan": gflop,
                        "fp64_tflops": gflop / statistics.median(times)}
    out["c4"] = run_update_c4(torch, steps)
    return out, model, kernel


def run_update_c4(torch, steps=5):
    """C4: M = 65,536 centres (256 x 256 lattice, bumps terrain, selected from
    10^6 support points); per-scan update with 20k points in a 2.5 m footprint."""
    from paper_2509_26222_b200 import terrain as T
    rng = np.random.default_rng(4)
    side = 17.85
    sup = rng.uniform(0.0, side, size=(1_000_000, 2))
    cs = T.select_centers(T.TerrainObservation(sup, terrain_c5(sup[:, 0], sup[:, 1], np)),
                          T.Rect((0.0, 0.0), (side, side)), RES, R_A, COUNT)
    kernel = T.KernelParams()
    kernel.finalize()
    model = T.TerrainModel(kernel, cs)

    def scan(cx, cy, m=20000):
        r = 2.5 * np.sqrt(rng.uniform(0, 1, m))
        a = rng.uniform(0, 2 * np.pi, m)
        clean = np.stack([cx + r * np.cos(a), cy + r * np.sin(a)], 1)
        noisy = clean + rng.normal(0.0, 0.02, size=(m, 2))
        return T.TerrainObservation(np.ascontiguousarray(noisy),
                                    terrain_c5(clean[:, 0], clean[:, 1], np))

    scans = [scan(4.0 + 0.5 * k, 8.0 + 0.3 * k) for k in range(steps + 2)]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for k, s in enumerate(scans):
        ev0.record()
        rep = model.recursive_update(s, False)
        ev1.record()
        ev1.synchronize()
        if k >= 2:
            times.append(ev0.elapsed_time(ev1))
    out = {"M": model.num_centers(), "m": 20000, "footprint_m": 2.5,
           "ms_per_scan": statistics.median(times), "ms_min": min(times),
           "gflop_per_scan": rep.flops / 1e9,
           "fp64_tflops": rep.flops / 1e9 / statistics.median(times),
           "n_active": rep.active_centers, "active_blocks": rep.active_blocks,
           "solver": rep.solver, "rejected": rep.rejected}
    # fit_batch_ridge at C4 scale (terrain_model.cpp:269-308):
    # banded Gram / Cholesky / solve over the 10^6 support points
    obs = T.TerrainObservation(sup, terrain_c5(sup[:, 0], sup[:, 1], np))
    T.fit_batch_ridge(kernel, cs, obs)
    fit_ms = []
    for _ in range(3):  # each call builds its model (device allocations): median of 3
        ev0.record()
        T.fit_batch_ridge(kernel, cs, obs)
        ev1.record()
        ev1.synchronize()
        fit_ms.append(ev0.elapsed_time(ev1))
    out["batch_fit_ms"] = statistics.median(fit_ms)
    out["batch_fit_ms_runs"] = fit_ms
    out["batch_fit_points"] = len(sup)
    return out


def run_batch_fit_c5(torch, device, rank, world, n_total=10_000_000, seed=11):
    """C5 kernel-matrix assembly + batch ridge, point-sharded (SURVEY §8d C5,
    §8e): the 316 x 316 lattice (99,856 centres) on every rank, n_total
    points split over the ranks (strong scaling), banded partial systems
    summed with one NCCL all-reduce each for H and b, every rank solving.
    CUDA-event times per phase, max over ranks."""
    import torch.distributed as dist
    from paper_2509_26222_b200 import terrain as T
    side = ROI_C5[1][0]
    nodes = np.arange(int(round(side / RES)) + 1) * RES
    gx, gy = np.meshgrid(nodes, nodes, indexing="ij")
    cs = T.CenterSet(np.stack([gx.ravel(), gy.ravel()], 1), RES, R_A, COUNT, T.Rect(*ROI_C5))
    kernel = T.KernelParams()
    kernel.finalize()
    model = T.TerrainModel(kernel, cs)
    n, ld, elems = model.batch_system()
    base, extra = divmod(n_total, world)
    m = base + (1 if rank < extra else 0)
    g = torch.Generator(device=f"cuda:{device}").manual_seed(seed + rank)
    xy = torch.rand((m, 2), generator=g, device=f"cuda:{device}", dtype=torch.float64) * side
    z = terrain_c5(xy[:, 0], xy[:, 1], torch)
    H = torch.empty(elems, dtype=torch.float64, device=f"cuda:{device}")
    b = torch.empty(n, dtype=torch.float64, device=f"cuda:{device}")
    nnz = model.batch_pattern()
    P = torch.empty(nnz, dtype=torch.float64, device=f"cuda:{device}") if world > 1 else None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    times = []
    for it in range(2):  # warm-up (workspaces, NCCL channels), then timed
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev[0].record()
        model.batch_assemble(xy, z, H, b, add_lambda=(rank == 0))
        ev[1].record()
        if world > 1:  # the structural nonzeros only (distributed.fit_batch_ridge_sharded)
            model.batch_pack(H, P)
            dist.all_reduce(P)
            model.batch_unpack(P, H)
            dist.all_reduce(b)
        ev[2].record()
        model.batch_solve(H, b)
        ev[3].record()
        torch.cuda.synchronize()
        times = [ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3]),
                 ev[0].elapsed_time(ev[3])]
    if world > 1:
        t = torch.tensor(times, dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times = t.tolist()
    q = torch.rand((20000, 2), generator=g, device=f"cuda:{device}", dtype=torch.float64)
    q = q * (side - 1.0) + 0.5
    zq, s, _, _ = model.predict(q, gradient=False)
    err = (zq - terrain_c5(q[:, 0], q[:, 1], torch)).abs()[s.bool()]
    return {"centres": n, "points_total": n_total, "points_per_rank": m, "band_ld": ld,
            "system_gb": elems * 8 / 1e9, "reduced_gb": (nnz + n) * 8 / 1e9,
            "assemble_ms": times[0], "allreduce_ms": times[1],
            "solve_ms": times[2], "total_ms": times[3], "scaling": "strong",
            "fit_abs_err_median": float(err.median()),
            "timing": "CUDA events per phase, max over ranks; the all-reduce phase packs the "
                      "band's structural nonzeros, reduces them and unpacks; solve replicated on "
                      "every rank"}


def match_scene(seed, n):
    """Synthetic LiDAR features: ground plane, two walls, three poles (edge
    features), labelled, in random order."""
    rng = np.random.default_rng(seed)
    g = np.c_[rng.uniform(-5, 5, n), rng.uniform(-5, 5, n), rng.normal(0, 0.004, n)]
    w1 = np.c_[np.full(n // 2, 3.0) + rng.normal(0, 0.004, n // 2), rng.uniform(-5, 5, n // 2),
               rng.uniform(0, 2.5, n // 2)]
    w2 = np.c_[rng.uniform(-5, 3, n // 2), np.full(n // 2, 4.0) + rng.normal(0, 0.004, n // 2),
               rng.uniform(0, 2.5, n // 2)]
    poles = [np.c_[np.full(300, x), np.full(300, y), rng.uniform(0, 2.5, 300)] +
             rng.normal(0, 0.002, (300, 3)) for x, y in [(1.0, 1.0), (-2.0, 0.5), (0.5, -3.0)]]
    e = np.concatenate(poles)
    P = np.concatenate([g, w1, w2, e])
    K = np.concatenate([np.full(len(g), 2), np.ones(len(w1) + len(w2)), np.zeros(len(e))])
    L = np.concatenate([np.zeros(len(g)), np.full(len(w1), 1), np.full(len(w2), 2),
                        np.repeat([3, 4, 5], 300)])
    perm = rng.permutation(len(P))
    return P[perm], K[perm].astype(np.uint8), L[perm].astype(np.int32)


def run_match_bench(torch, cpu=True, steps=10):
    """association of a ~17k-feature scan against a 20-frame
    LocalMap (~240k map points): build_correspondences + feature normal
    equations per LM outer iteration; the reference algorithm (restated
    kd-tree, one core) beside it."""
    from paper_2509_26222_b200 import match as Mt
    gm = Mt.LocalMap(0.1, 20)
    om = None
    if cpu:
        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle as orc
        om = orc.LocalMap(0.1, 20)
    for f in range(20):
        P, K, L = match_scene(100 + f, 8000)
        R = so3_exp(np.array([0.0, 0.0, 0.01 * f]))
        t = np.array([0.02 * f, 0.0, 0.0])
        Ps = (P - t) @ R
        gm.insert(Ps, K, L, R, t)
        if om is not None:
            om.insert(Ps, K, L, R, t)
    P, K, _ = match_scene(7, 8000)
    R = so3_exp(np.array([0.002, -0.001, 0.2]))
    t = np.array([0.4, -0.1, 0.0])
    Ps = (P - t) @ R + np.random.default_rng(3).normal(0, 0.01, P.shape)
    Mt.build_correspondences(Ps, K, R, t, gm)
    Mt.feature_normal_eq(gm, R, t)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        c = Mt.build_correspondences(Ps, K, R, t, gm)
    t1 = time.perf_counter()
    for _ in range(steps):
        Mt.feature_normal_eq(gm, R, t)
    t2 = time.perf_counter()
    out = {"map_points": gm.size(), "features": len(P), "correspondences": len(c),
           "associate_ms": (t1 - t0) / steps * 1e3, "feature_ne_ms": (t2 - t1) / steps * 1e3,
           "timing": "wall clock per call through the Python API (host features in, "
                     "host correspondences out)"}
    if om is not None:
        t3 = time.perf_counter()
        o = om.build_correspondences(Ps, K, R, t)
        out["cpu_reference_associate_ms"] = (time.perf_counter() - t3) * 1e3
        out["cpu_reference"] = "oracle restatement of scan_matcher.cpp:44-183 with the kd-tree, 1 core"
        out["cpu_correspondences"] = len(o["kind"])
    return out


def run_consumers_bench(torch, umodel, ukernel, cpu=True, reps=10):
    """SURVEY §8f row 4 consumers through the Python API, host arrays in and
    out (wall clock per call): select_ground_points on a 200k-feature scan,
    terrain_error_histogram on 10^6 samples against the C3 model; the oracle
    restatements (one core) beside them."""
    from paper_2509_26222_b200 import consumers as K
    from paper_2509_26222_b200 import terrain as T
    rng = np.random.default_rng(21)
    n = 200_000
    p = np.c_[rng.uniform(-4, 4, n), rng.uniform(-4, 4, n), rng.normal(0, 0.02, n)]
    kinds = rng.choice(np.array([0, 1, 2], dtype=np.uint8), n, p=[0.1, 0.3, 0.6])
    R = so3_exp(np.array([0.01, 0.02, 0.7]))
    t = np.array([2.2, 2.2, 0.4])
    roi = T.Rect((0.0, 0.0), (4.41, 4.41))
    K.select_ground_points(p, kinds, R, t, roi, 2.5, 0.12, 20000)
    t0 = time.perf_counter()
    for _ in range(reps):
        obs = K.select_ground_points(p, kinds, R, t, roi, 2.5, 0.12, 20000)
    sel_ms = (time.perf_counter() - t0) / reps * 1e3
    m = 1_000_000
    xy = rng.uniform(0.0, 4.41, (m, 2))
    z = staircase(xy[:, 0]) + rng.normal(0.0, 0.01, m)
    K.terrain_error_histogram(umodel, xy, z, 0.05, 25)
    t0 = time.perf_counter()
    for _ in range(reps):
        h = K.terrain_error_histogram(umodel, xy, z, 0.05, 25)
    hist_ms = (time.perf_counter() - t0) / reps * 1e3
    # RBFT snapshot round trip of the C3 model (§8f row 3; byte layout of
    # snapshot.cpp:7-126, tests/test_gpu_parity.py checks the bytes)
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        path = str(Path(td) / "c3.rbft")
        umodel.save(path)
        T.TerrainModel.load(path)  # warm-up (workspaces, module loading)
        t0 = time.perf_counter()
        umodel.save(path)
        save_ms = (time.perf_counter() - t0) * 1e3
        t0 = time.perf_counter()
        T.TerrainModel.load(path)
        load_ms = (time.perf_counter() - t0) * 1e3
        snap_bytes = Path(path).stat().st_size
    out = {"snapshot_bytes": snap_bytes, "snapshot_save_ms": save_ms, "snapshot_load_ms": load_ms,
           "ground_scan_points": n, "ground_kept": len(obs.z), "select_ground_ms": sel_ms,
           "histogram_samples": m, "histogram_ms": hist_ms, "histogram_total": h.total(),
           "timing": "wall clock per call through the Python API (host arrays in/out)"}
    if cpu:
        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle as orc
        t0 = time.perf_counter()
        orc.select_ground_points(p, kinds, R, t, roi, 2.5, 0.12, 20000)
        out["cpu_reference_select_ground_ms"] = (time.perf_counter() - t0) * 1e3
        om = orc.Model(ukernel, umodel.centers())
        om.set_weights(umodel.weights())
        ms = 100_000
        t0 = time.perf_counter()
        om.error_histogram(xy[:ms], z[:ms], 0.05, 25)
        out["cpu_reference_histogram_ms_per_1e6"] = (time.perf_counter() - t0) * 1e3 * (m / ms)
        out["cpu_reference"] = "oracle restatements (pipeline.cpp:150-170, metrics.cpp:199-232), 1 core"
    return out


def cpu_update_ms(model, kernel, m=400, seed=5):
    """The reference's recursive_update (chunk-64 Woodbury; its GEMMs on all
    host threads) at M = 4096 from the GPU model's weights."""
    orc, _ = cpu_backend()
    cs = model.centers()
    om = orc.Model(kernel, cs)
    om.set_weights(model.weights())
    rng = np.random.default_rng(seed)
    clean = rng.uniform(0.0, 4.41, size=(m, 2))
    noisy = clean + rng.normal(0.0, 0.1, size=(m, 2))
    t0 = time.perf_counter()
    rep = om.recursive_update(noisy, staircase(clean[:, 0]))
    return (time.perf_counter() - t0) * 1e3, rep


def c5_parity(model, kernel, cs, w, R, tv, h, n=100_000):
    """Self-check of the measured kernel (cpu_baseline leg): k_manifold on the
    first n C5 lever arms vs the reference's manifold rows with the same
    weights, at the SURVEY §8d tolerance: |d| <= 1e-9 max(|ref|, scale) with
    the row's sum |w kappa| scale (no additive floor)."""
    from paper_2509_26222_b200 import kinematics as kin
    from paper_2509_26222_b200.terrain import CenterSet, Rect
    orc, kind = cpu_backend()
    hs = np.ascontiguousarray(np.stack([x[:n].cpu().numpy() for x in h], 1))
    rows, _ = kin.manifold_rows(model, R, tv, tuple(np.ascontiguousarray(hs[:, j]) for j in range(3)),
                                0.0, 1.0, 0.05, want=("r", "J", "valid"))
    om = orc.Model(kernel, CenterSet(cs.centers, RES, R_A, COUNT, Rect(*ROI_C5)))
    om.set_weights(w)
    ref, _ = om.manifold_rows(R, tv, hs, 0.0, 1.0, 0.05, threads=os.cpu_count() or 1)
    xy = (hs @ np.asarray(R).T + tv)[:, :2]
    S0, S1 = om.scales(xy)
    s = np.abs(ref["J"][:, 5])
    hn = np.linalg.norm(hs, axis=1)
    J = rows["J"].reshape(6, -1).T
    tiny = np.finfo(np.float64).tiny
    scale_J = [s * hn * S1, s * hn * S1, s * hn * S1, s * S1, s * S1, s]

    def worst(got, want, scale):
        return float(np.max(np.abs(got - want) / np.maximum(np.maximum(np.abs(want), scale), tiny)))

    er = worst(rows["r"], ref["r"], s * S0)
    eJ = max(worst(J[:, c], ref["J"][:, c], scale_J[c]) for c in range(6))
    vm = int(np.sum(rows["valid"] != ref["valid"]))
    return {"points": n, "source": kind, "kernel_kind": int(model.sweep()[0]),
            "max_err_r": er, "max_err_J": eJ, "valid_mismatch": vm,
            "tolerance": 1e-9, "pass": bool(er <= 1e-9 and eJ <= 1e-9 and vm == 0),
            "scale": "1e-9 * max(|ref|, s sum|w kappa| [r], s |h| sum|w kappa| d/sigma^2 [J_rot], "
                     "s sum|w kappa| d/sigma^2 [J_t])"}


def c1_inputs_np(n_points=20000, seed=2509):
    """20k points uniform on [0, 1.05]^2 with N(0, 0.1^2) xy
    noise, z = 0.1 sin 4x + 0.05 y^2 of the clean point."""
    rng = np.random.default_rng(seed)
    clean = rng.uniform(0.0, 1.05, (n_points, 2))
    noisy = clean + rng.normal(0.0, 0.1, clean.shape)
    z = 0.1 * np.sin(4.0 * clean[:, 0]) + 0.05 * clean[:, 1] ** 2
    return np.ascontiguousarray(noisy), z


def run_c1(torch, cpu=True):
    """C1 (BASELINE configs[0]): M = 256 centres on [0, 1.05]^2, one 20k-point
    scan: select_centers, one recursive_update (n = 256, m = 20k) and the
    height / gradient / manifold-row evaluation of the scan, each timed on
    the GPU (CUDA events, host arrays through the public API) and on the
    CPU with the reference (oracle/_ref, all host threads)."""
    from paper_2509_26222_b200 import kinematics as kin
    from paper_2509_26222_b200 import terrain as T
    xy, z = c1_inputs_np()
    roi = T.Rect((0.0, 0.0), (1.05, 1.05))
    R, tv = so3_exp(POSE_W), np.array(POSE_T)
    P = np.concatenate([xy, z[:, None]], 1)
    H = (P - tv) @ R
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(f, reps=5):
        f()
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            ev0.record()
            out = f()
            ev1.record()
            ev1.synchronize()
            ts.append(ev0.elapsed_time(ev1))
        return statistics.median(ts), out

    obs = T.TerrainObservation(xy, z)
    k = T.KernelParams()
    k.finalize()
    sel_ms, cs = timed(lambda: T.select_centers(obs, roi, RES, R_A, COUNT))

    def upd():
        m = T.TerrainModel(k, cs)
        return m, m.recursive_update(obs, False)
    upd_ms, (model, rep) = timed(upd)
    eval_ms, _ = timed(lambda: model.predict(xy))
    rows_ms, _ = timed(lambda: kin.manifold_rows(model, R, tv, H, 0.0, 1.0, 0.05))
    out = {"M": len(cs.centers), "m": len(z), "n_active": rep.active_centers, "solver": rep.solver,
           "gpu_ms": {"select_centers": sel_ms, "model_and_recursive_update": upd_ms,
                      "predict_height_gradient": eval_ms, "manifold_rows_normal_eq": rows_ms}}
    if cpu:
        orc, kind = cpu_backend()
        th = os.cpu_count() or 1
        t0 = time.perf_counter()
        nodes = orc.supported_mesh_nodes(xy, z, roi, RES, R_A, COUNT, True)
        t1 = time.perf_counter()
        om = orc.Model(k, T.CenterSet(nodes, RES, R_A, COUNT, roi))
        om.recursive_update(xy, z, False)
        t2 = time.perf_counter()
        om.predict(xy, threads=1)
        t3 = time.perf_counter()
        om.manifold_rows(R, tv, H, 0.0, 1.0, 0.05, threads=1)
        t4 = time.perf_counter()
        out["cpu_ms"] = {"select_centers": (t1 - t0) * 1e3, "model_and_recursive_update": (t2 - t1) * 1e3,
                         "predict_height_gradient": (t3 - t2) * 1e3,
                         "manifold_rows_normal_eq": (t4 - t3) * 1e3}
        out["cpu"] = {"kind": kind, "cores": th,
                      "note": "update on all host threads (GEMMs of the compiled reference); "
                              "evaluation single-threaded like the reference's per-query path"}
        out["nodes_bit_exact_vs_cpu"] = bool(np.array_equal(np.asarray(cs.centers).view(np.uint64),
                                                          nodes.view(np.uint64)))
    return out


def cpu_reference_figures(torch):
    """CPU figures beside the GPU's at reduced sizes the CPU reference
    finishes in seconds (its dense chunk-64 Woodbury is 4 n^2 m flops):
    C3-reduced (M = 400 staircase lattice, m = 20,000: the information form on
    the GPU) and C4-reduced (97 x 97 bumps lattice, a 1 m footprint,
    m = 2,000). Same inputs on both; ms per update and the weights' relative
    difference."""
    from paper_2509_26222_b200 import terrain as T
    orc, kind = cpu_backend()
    k = T.KernelParams()
    k.finalize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {"kind": kind, "cores": os.cpu_count() or 1}

    def lattice(side, seed):
        roi = T.Rect((0.0, 0.0), (side, side))
        rng = np.random.default_rng(seed)
        sup = rng.uniform(0.0, side, (int(side * side * 1500), 2))
        return T.select_centers(T.TerrainObservation(sup, np.zeros(len(sup))), roi, RES, R_A, COUNT)

    rng = np.random.default_rng(41)
    cases = []
    cs3 = lattice(1.33, 1)
    clean = rng.uniform(0.0, 1.33, (20000, 2))
    cases.append(("c3_reduced_m20000", cs3, clean + rng.normal(0.0, 0.1, clean.shape),
                  staircase(clean[:, 0] + 0.4)))
    cs4 = lattice(6.72, 6)
    rr = np.sqrt(rng.uniform(0, 1, 2000))
    a = rng.uniform(0, 2 * np.pi, 2000)
    clean = np.stack([3.0 + rr * np.cos(a), 3.2 + rr * np.sin(a)], 1)
    cases.append(("c4_reduced_m2000", cs4, clean + rng.normal(0.0, 0.02, clean.shape),
                  terrain_c5(clean[:, 0], clean[:, 1], np)))
    for name, cs, xy, z in cases:
        g = T.TerrainModel(k, cs)
        g.recursive_update(T.TerrainObservation(xy, z), False)  # warm
        g = T.TerrainModel(k, cs)
        torch.cuda.synchronize()
        ev0.record()
        rep = g.recursive_update(T.TerrainObservation(xy, z), False)
        ev1.record()
        ev1.synchronize()
        om = orc.Model(k, cs)
        t0 = time.perf_counter()
        om.recursive_update(xy, z, False)
        cpu_ms = (time.perf_counter() - t0) * 1e3
        wr = om.weights()
        out[name] = {"M": len(cs.centers), "m": len(z), "n_active": rep.active_centers,
                     "solver": rep.solver, "gpu_ms": ev0.elapsed_time(ev1), "cpu_ms": cpu_ms,
                     "weights_rel_diff": float(np.linalg.norm(g.weights() - wr) / np.linalg.norm(wr))}
    return out


def reference_c2(scans=20):
    """The reference's own pipeline::run_odometry (oracle/_ref) on its stock
    staircase simulation at 1000 x 20 rays, RunConfig
    defaults with use_imu false (the GPU loop's prediction): per-scan wall
    time on the host. The GPU loop on the same bundle is compared pose by pose
    in tests/test_pose_parity.py (profiles/r2_pose_parity.jsonl)."""
    orc, kind = cpu_backend()
    if kind != "reference":
        return {"unavailable": "oracle/_ref not built"}
    b = orc.SimBundle("staircase", 11, 1000, 20, scans)
    o = orc.odometry(b, orc.run_config_json(use_imu=False), mode=1)
    feats = float(np.mean([len(b.scan(k)[1]) for k in range(b.num_scans())]))
    return {"kind": kind, "scans": int(b.num_scans()), "features_per_scan": feats,
            "ms_per_scan_median": float(np.median(o["wall_ms"][1:])),
            "ms_per_scan_mean": float(np.mean(o["wall_ms"][1:])), "threads": 1}


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--points", type=int, default=10_000_000)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-update", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    # one process per GPU: `--gpus N` without a torchrun environment launches
    # N ranks itself (torch.distributed.run on 127.0.0.1); under torchrun the
    # world size must agree with --gpus
    if os.environ.get("WORLD_SIZE") is None and args.gpus > 1:
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}")

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    from paper_2509_26222_b200 import distributed as D
    from paper_2509_26222_b200 import kinematics as kin
    from paper_2509_26222_b200 import terrain as T

    ctx = T.Context.default(local)
    model, kernel, cs, w, R, tv, h = build_c5(local, args.points, 1000 + rank, torch)
    n = args.points
    rows = {"r": torch.empty(n, dtype=torch.float64, device="cuda"),
            "J": torch.empty(6 * n, dtype=torch.float64, device="cuda"),
            "valid": torch.empty(n, dtype=torch.uint8, device="cuda")}
    ne_buf = torch.zeros(29, dtype=torch.float64, device="cuda")
    # bin the scan once under a perturbed initial-guess pose (LM re-evaluates
    # the same scan every iteration; the binning is amortised over them)
    R0 = so3_exp(np.array(POSE_W) + np.array([0.004, -0.003, 0.01]))
    kin.Scan(model, R0, tv, h)  # first binning also sizes the workspace (not timed)
    scan = kin.Scan(model, R0, tv + np.array([0.03, -0.02, 0.01]), h)
    bin_ms = scan.bin_ms()

    def step():
        _, ne = scan.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rows)
        if world > 1:  # NCCL: the 29-double normal-equation reduce
            ne = D.allreduce_normal_eq(ne, buf=ne_buf)
        return ne

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    lib = __import__("paper_2509_26222_b200._abi", fromlist=["load"]).load()
    import ctypes as C
    lib.tlg_ctx_set_profiling(ctx.handle, 1)
    l0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(args.steps):
            ne = step()
        ev1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    launches = ctx.launch_count() - l0
    kms, kn = C.c_double(), C.c_uint64()
    lib.tlg_ctx_kernel_stats(ctx.handle, 0, C.byref(kms), C.byref(kn))
    lib.tlg_ctx_set_profiling(ctx.handle, 0)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = world * n / (ms_step * 1e-3)
    k_ms = kms.value / max(1, kn.value)

    # ---- e2e: host (pinned) lever arms in, normal equations out ------------
    hh = [torch.empty(n, dtype=torch.float64, pin_memory=True) for _ in range(3)]
    for j in range(3):
        hh[j].copy_(h[j])
    hn = tuple(x.numpy() for x in hh)
    # the rows are materialised on the device exactly as in `value` (r, J,
    # valid); only the normal equations come back to the host
    for _ in range(2):
        kin.manifold_rows(model, R, tv, hn, 0.0, 1.0, 0.05, out=rows)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(3, min(args.steps, 10))
    e0.record()
    for _ in range(e2e_steps):
        kin.manifold_rows(model, R, tv, hn, 0.0, 1.0, 0.05, out=rows)
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    del hh, hn

    peaks, peak_kind = load_peaks()
    achieved = BYTES_PER_POINT * n / (k_ms * 1e-3) / 1e9
    traffic, ncu_info = None, {}
    tf = ROOT / "profiles" / "kernel_traffic.json"
    if tf.exists():
        try:
            d = json.loads(tf.read_text())
            if d.get("k_manifold", {}).get("points") == n:
                traffic = d["k_manifold"]["dram_bytes_per_launch"]
                ncu_info = {"fp64_pipe_pct_ncu": d["k_manifold"].get("fp64_pipe_pct_active"),
                            "issue_active_pct_ncu": d["k_manifold"].get("issue_active_pct"),
                            "l1_lsu_wavefronts_pct_ncu":
                                d["k_manifold"].get("l1_lsu_wavefronts_pct_elapsed")}
        except Exception:
            traffic = None
    # point-centre pairs within the cutoff (the reference's centers_near), on
    # a 200k-point sample of the workload: pairs/s beside points/s
    ns = min(n, 200_000)
    hs = np.stack([hh_.cpu().numpy() for hh_ in (h[0][:ns], h[1][:ns], h[2][:ns])], 1)
    xw = hs @ np.asarray(R).T + np.asarray(tv)
    rp, _, _ = model.moment_features(np.ascontiguousarray(xw[:, :2]))
    pairs_per_point = float(rp[-1]) / ns

    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C5: 1e7 LiDAR ground points/GPU x 99,856 RBF centres "
                               "(316x316 lattice, sigma=0.04, sigma_eps=0.1, cutoff 0.3231 m), "
                               "manifold rows r+J[6]+valid materialised + fused J^T J/J^T r/cost",
                   "points_per_gpu": n, "centres": len(cs.centers), "parallelism": f"dp{world}",
                   "l2": "inputs (240 MB/GPU) larger than L2; no flush",
                   "step": "one LM cost evaluation (tlg_scan_manifold_rows) over a scan binned "
                           "once under a perturbed initial pose",
                   "scan_bin_ms": bin_ms},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic,
                     "kernel": "k_manifold", "kernel_ms": k_ms,
                     "bytes_per_point": BYTES_PER_POINT, "peak_source": peak_kind,
                     "pairs_per_point": pairs_per_point,
                     "pairs_per_s": world * n / (k_ms * 1e-3) * pairs_per_point,
                     "binding": "FP64 issue latency and L1 window gathers (ncu), not HBM",
                     **ncu_info},
        "e2e": {"value": world * n / (e2e_ms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": 24 * n, "d2h_bytes_per_step": 29 * 8 + 4,
                "ms_per_step": e2e_ms, "api": "tlg_manifold_rows, pinned host lever arms in, rows r/J/valid "
                                              "materialised in HBM, normal equations out"},
        "clocks": clk.summary(),
    }

    if not args.no_update:
        # C5 kernel-matrix assembly + batch ridge, point-sharded over the ranks
        # (collective: every rank runs it)
        result["batch_fit_c5"] = run_batch_fit_c5(torch, local, rank, world)
    if rank == 0 and world == 1:
        dfma, dmma = C.c_double(), C.c_double()
        __import__("paper_2509_26222_b200._abi", fromlist=["load_diag"]).load_diag().tlg_diag_fp64_peak(
            ctx.handle, C.byref(dfma), C.byref(dmma))
        result["fp64_peak_tflops"] = {"dfma": dfma.value, "dmma": dmma.value}
        # FP64 view of the same kernel (pairs/s based)
        if not args.no_update:
            upd, umodel, ukernel = run_update_bench(torch, local)
            # F / t / P_FP64: the formulation's flops over the
            # measured DMMA peak of this run
            for key in ("m400", "m20000", "c4"):
                if key in upd and "fp64_tflops" in upd[key]:
                    upd[key]["dmma_peak_frac"] = upd[key]["fp64_tflops"] / dmma.value
            result["update"] = upd
            if not args.no_cpu:
                cms, crep = cpu_update_ms(umodel, ukernel, 400)
                result["update"]["cpu_ms_per_scan_m400"] = cms
                result["update"]["cpu_n_active"] = crep["active_centers"]
                result["update"]["cpu_kind"] = cpu_backend()[1]
        if not args.no_update:
            result["match"] = run_match_bench(torch, not args.no_cpu)
            result["consumers"] = run_consumers_bench(torch, umodel, ukernel, not args.no_cpu)
            # C2-style odometry stream (BASELINE configs[1]): the restated
            # pipeline.cpp:196-300 loop over synthetic staircase scans
            sys.path.insert(0, str(ROOT / "tools"))
            from pipeline_c2 import run_c2
            c2 = run_c2(scans=100)
            c2["note"] = ("synthetic staircase with walls and poles, ~20k features/scan; host "
                          "(Python) LM loop over device association, rows and update")
            result["pipeline_c2"] = c2
            result["c1"] = run_c1(torch, cpu=not args.no_cpu)
        if not args.no_cpu:
            # ---- cpu_baseline leg: the reference on the host cores, and the
            # checks that use it (parity of the measured kernel) -------------
            _, kind = cpu_backend()
            pts_h = torch.stack(list(h), 1)[: 2_000_000].cpu().numpy()
            rate, ns, threads, dt, _ = cpu_eval_rate(cs.centers, w, kernel, pts_h, R, tv,
                                                     args.cpu_seconds)
            what = ("the reference compiled from its unchanged sources (oracle/_ref)"
                    if kind == "reference" else "oracle restatement -O3 no-FMA")
            result["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads,
                                      "kind": kind,
                                      "sample": f"{ns} of the C5 points ({dt:.1f} s), {what}, "
                                                f"{threads} threads over points"}
            result["parity"] = c5_parity(model, kernel, cs, w, R, tv, h)
            if not args.no_update:
                result["update"]["cpu_reference"] = cpu_reference_figures(torch)
                result["pipeline_c2"]["reference_c2"] = reference_c2(20)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU path (oracle/_ref, its
    unchanged sources compiled against a minimal Eigen subset; the
    restatement if that is absent) on the host cores, same metric."""
    if rank != 0:
        return
    import torch
    from paper_2509_26222_b200 import terrain as T  # noqa: F401  (types only)
    sys.path.insert(0, str(ROOT / "oracle"))
    rng = np.random.default_rng(1000)
    # C5 model: full 316 x 316 lattice (what select_centers yields at 1e6 support points)
    nx = int(math.floor(22.05 / RES + 1e-9))
    ii, jj = np.meshgrid(np.arange(nx + 1), np.arange(nx + 1), indexing="ij")
    centers = np.stack([0.0 + ii.ravel() * RES, 0.0 + jj.ravel() * RES], 1)
    kernel = T.KernelParams()
    kernel.cutoff_radius = 3.0 * kernel.sigma_tilde()
    w = terrain_c5(centers[:, 0], centers[:, 1], np) * RES * RES / (2 * math.pi * kernel.sigma ** 2)
    R, tv = so3_exp(POSE_W), np.array(POSE_T)
    m = 2_000_000
    p = rng.uniform(0.0, 22.05, size=(m, 2))
    pz = terrain_c5(p[:, 0], p[:, 1], np) + 0.01 * rng.normal(size=m)
    H = (np.stack([p[:, 0], p[:, 1], pz], 1) - tv) @ R
    threads = os.cpu_count() or 1
    per_step = max(2.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    _, kind = cpu_backend()
    rate, ns, threads, dt, om = cpu_eval_rate(centers, w, kernel, H, R, tv, per_step, threads)
    rates = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        om.manifold_rows(R, tv, H[:ns], 0.0, 1.0, 0.05, threads=threads)
        d = time.perf_counter() - t0
        if i >= args.warmup:
            rates.append(ns / d)
    value = statistics.median(rates)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ns / value * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": {"workload": "C5 (bounded sample per step)", "points_per_step": ns,
                      "centres": len(centers)},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                            "sample": f"{ns} C5 points per step; "
                                      + ("the reference compiled from its unchanged sources "
                                         "(oracle/_ref: minimal Eigen subset in place of Eigen3)"
                                         if kind == "reference" else
                                         "oracle restatement of the reference")},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
