"""Association throughput: LocalMap of 20 frames x 20k
features, build_correspondences + feature normal equations for a 20k-feature
scan, device vs the oracle restatement on one host core."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import oracle as orc  # noqa: E402
from paper_2509_26222_b200 import match as M  # noqa: E402
from test_match import _scene  # noqa: E402


def main():
    gm, om = M.LocalMap(0.1, 20), orc.LocalMap(0.1, 20)
    for f in range(20):
        P, K, L = _scene(100 + f, 8000)
        R = orc.so3_exp([0.0, 0.0, 0.01 * f])
        t = np.array([0.02 * f, 0.0, 0.0])
        Ps = (P - t) @ R
        gm.insert(Ps, K, L, R, t)
        if "--cpu" in sys.argv:
            om.insert(Ps, K, L, R, t)
    P, K, _ = _scene(7, 8000)
    R = orc.so3_exp([0.002, -0.001, 0.2])
    t = np.array([0.4, -0.1, 0.0])
    Ps = (P - t) @ R + np.random.default_rng(3).normal(0, 0.01, P.shape)
    M.build_correspondences(Ps, K, R, t, gm)
    t0 = time.perf_counter()
    reps = 10
    for _ in range(reps):
        c = M.build_correspondences(Ps, K, R, t, gm)
    t1 = time.perf_counter()
    for _ in range(reps):
        ne = M.feature_normal_eq(gm, R, t)
    t2 = time.perf_counter()
    print(f"map {gm.size()} pts; scan {len(P)} features -> {len(c)} correspondences: "
          f"associate {(t1 - t0) / reps * 1e3:.2f} ms, feature NE {(t2 - t1) / reps * 1e3:.3f} ms "
          f"(wall, incl. host<->device copies)", flush=True)
    if "--cpu" in sys.argv:
        t3 = time.perf_counter()
        o = om.build_correspondences(Ps, K, R, t)
        t4 = time.perf_counter()
        print(f"oracle (1 core): associate {(t4 - t3) * 1e3:.1f} ms -> {len(o['kind'])}", flush=True)


if __name__ == "__main__":
    main()
