"""C2-style odometry run: 100 scans x ~20k synthetic LiDAR
features over a staircase (0.08 m risers every 0.5 m) with walls and poles,
run through paper_2509_26222_b200.pipeline.run_odometry (lm_solve with feature
+ wheel manifold rows, map insert, ground selection, terrain update with
births). Prints per-stage wall time per scan and the trajectory error."""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2509_26222_b200 import match as M  # noqa: E402
from paper_2509_26222_b200 import pipeline as PL  # noqa: E402
from paper_2509_26222_b200 import terrain as T  # noqa: E402


def stairs(x):
    return 0.08 * np.floor(np.clip(x, 0.0, None) / 0.5)


def make_scan(rng, R, t, n=20000, rng_m=6.0):
    ng, nw, npl = int(n * 0.7), int(n * 0.25), n - int(n * 0.7) - int(n * 0.25)
    r = rng_m * np.sqrt(rng.uniform(0.02, 1.0, ng))
    a = rng.uniform(0, 2 * np.pi, ng)
    gx, gy = t[0] + r * np.cos(a), t[1] + r * np.sin(a)
    G = np.c_[gx, gy, stairs(gx) + rng.normal(0, 0.003, ng)]
    side = rng.integers(0, 2, nw)
    wx = t[0] + rng.uniform(-rng_m, rng_m, nw)
    W = np.c_[wx, np.where(side == 0, -3.0, 3.0) + rng.normal(0, 0.003, nw),
              stairs(wx) + rng.uniform(0, 2.0, nw)]
    poles = np.array([[px, py] for px in np.arange(0.7, 12, 1.7) for py in (-1.8, 1.9)])
    pid = rng.integers(0, len(poles), npl)
    E = np.c_[poles[pid] + rng.normal(0, 0.003, (npl, 2)), rng.uniform(0, 2.0, npl)]
    E[:, 2] += stairs(E[:, 0])
    P = np.concatenate([G, W, E])
    K = np.concatenate([np.full(ng, 2), np.ones(nw), np.zeros(npl)]).astype(np.uint8)
    keep = np.linalg.norm(P[:, :2] - t[:2], axis=1) < rng_m
    P, K = P[keep], K[keep]
    perm = rng.permutation(len(P))
    return ((P[perm] - t) @ R), K[perm]


def run_c2(scans=100, points=20000, manifold=True, verbose=False):
    """The C2-style run; returns a summary dict (also used by bench.py)."""
    a = argparse.Namespace(scans=scans, points=points, no_manifold=not manifold)
    rng = np.random.default_rng(11)
    dt = 0.1
    gt = []
    for k in range(a.scans):
        x = 0.2 + 0.05 * k
        yaw = 0.05 * np.sin(0.2 * k)
        R = M.so3_exp([0.0, 0.0, yaw])
        y = 0.1 * np.sin(0.1 * k)
        # the wheels (0.2 m ahead of the base) stand on the tread below them:
        # base height = tread height under the wheel centres + 0.3 m
        xw = x + 0.2 * np.cos(yaw)
        gt.append((R, np.array([x, y, stairs(xw) + 0.3])))
    scans, kinds = zip(*[make_scan(rng, R, t, a.points) for R, t in gt])
    lever = np.array([[0.2, 0.15, -0.25], [0.2, -0.15, -0.25]])
    roi = T.Rect((-1.0, -3.0), (12.0, 3.0))
    t0 = time.perf_counter()
    cfg = PL.RunConfig(use_manifold=not a.no_manifold)
    res = PL.run_odometry(scans, kinds, [k * dt for k in range(a.scans)], gt[0][0], gt[0][1], roi,
                          lever_arms=lever, wheel_radius=0.05, config=cfg)
    wall = time.perf_counter() - t0
    err = np.array([np.linalg.norm(tr[1] - g[1]) for tr, g in zip(res.trajectory, gt)])
    stages = {}
    for f in res.frames[1:]:
        for k, v in f.ms.items():
            stages.setdefault(k, []).append(v)
    med = {k: float(np.median(v)) for k, v in stages.items()}
    mean = {k: float(np.mean(v)) for k, v in stages.items()}
    if verbose:
        for f, e in zip(res.frames, err):
            s = f.solve
            if s is not None:
                ev = (res.trajectory[f.index][1] - gt[f.index][1]) * 100
                print(f"  frame {f.index}: err {e*100:.1f} cm ({ev[0]:.1f},{ev[1]:.1f},{ev[2]:.1f}) corr {s.correspondence_count} "
                      f"iters {s.outer_iterations} acc {s.accepted_steps} deg {s.degenerate} "
                      f"eig {s.smallest_feature_eigenvalue:.3g} cost {s.cost_trace[0]:.4g}->{s.final_cost:.4g}")
    held = sum(f.held for f in res.frames)
    corr = np.median([f.solve.correspondence_count for f in res.frames[1:]])
    per_scan = [sum(f.ms.values()) for f in res.frames[1:]]
    return {"scans": a.scans, "features_per_scan": a.points, "manifold_rows": not a.no_manifold,
            "ms_per_scan_wall": wall / a.scans * 1e3,
            "ms_per_scan_median": float(np.median(per_scan)),
            "wall_note": "wall includes scan 0 (the first terrain build with ~all births)",
            "stage_median_ms": med,
            "stage_mean_ms": mean, "median_correspondences": float(corr), "held": int(held),
            "ate_rmse_cm": float(np.sqrt(np.mean(err ** 2)) * 100),
            "ate_max_cm": float(err.max() * 100), "terrain_centres": res.terrain.num_centers()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scans", type=int, default=100)
    ap.add_argument("--points", type=int, default=20000)
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--no-manifold", action="store_true")
    a = ap.parse_args()
    r = run_c2(a.scans, a.points, not a.no_manifold, a.verbose)
    med, mean = r["stage_median_ms"], r["stage_mean_ms"]
    print(f"{'features + wheel manifold rows' if r['manifold_rows'] else 'features only'}: "
          f"{r['scans']} scans x ~{r['features_per_scan']} features: "
          f"{r['ms_per_scan_median']:.1f} ms/scan median ({r['ms_per_scan_wall']:.1f} wall incl. scan 0) "
          f"(median / mean stage ms: {', '.join(f'{k} {v:.2f}/{mean[k]:.2f}' for k, v in med.items())}); "
          f"median correspondences {r['median_correspondences']:.0f}; held {r['held']}; "
          f"ATE rmse {r['ate_rmse_cm']:.2f} cm, max {r['ate_max_cm']:.2f} cm; "
          f"terrain centres {r['terrain_centres']}", flush=True)


if __name__ == "__main__":
    main()
