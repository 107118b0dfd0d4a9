"""fit_batch_ridge timing: C3 (64 x 64 lattice, 20k points) and C4 (256 x 256
lattice = 65,536 centres, 10^6 points; banded path, dense n x n storage)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2509_26222_b200 import terrain as T  # noqa: E402


def bumps(x, y):
    return 0.05 * np.sin(2 * np.pi * x / 1.5) * np.sin(2 * np.pi * y / 1.5)


def run(side, n_pts, label):
    rng = np.random.default_rng(9)
    xy = rng.uniform(0.0, side, size=(n_pts, 2))
    z = bumps(xy[:, 0], xy[:, 1])
    obs = T.TerrainObservation(xy, z)
    roi = T.Rect((0.0, 0.0), (side, side))
    cs = T.select_centers(obs, roi, 0.07, 0.12, 3)
    k = T.KernelParams()
    k.finalize()
    T.fit_batch_ridge(k, cs, obs)  # warm-up (workspace)
    t0 = time.perf_counter()
    model = T.fit_batch_ridge(k, cs, obs)
    dt = time.perf_counter() - t0
    q = rng.uniform(0.5, side - 0.5, size=(20000, 2))
    zq, s, _, _ = model.predict(q, gradient=False)
    err = np.abs(zq - bumps(q[:, 0], q[:, 1]))[s.astype(bool)]
    print(f"{label}: M = {len(cs.centers)}, m = {n_pts}: fit {dt * 1e3:.1f} ms; "
          f"|f - z| median {np.median(err):.2e} p99 {np.quantile(err, 0.99):.2e}", flush=True)


if __name__ == "__main__":
    run(4.41, 20000, "C3")
    if "--c4" in sys.argv:
        run(17.85, 1_000_000, "C4")
