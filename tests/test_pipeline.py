"""The per-scan odometry loop (pipeline.cpp:196-300) over the device
components: lm_solve (association + feature rows, optional wheel manifold
rows), map insert, ground selection and terrain update with births."""
import sys
from pathlib import Path

import numpy as np
import pytest

sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))


@pytest.mark.gpu
@pytest.mark.parametrize("manifold", [False, True])
def test_run_odometry_short(gpu_ctx, manifold):
    import pipeline_c2 as P
    from paper_2509_26222_b200 import pipeline as PL
    from paper_2509_26222_b200 import terrain as T
    rng = np.random.default_rng(11)
    gt = []
    for k in range(12):
        x = 0.2 + 0.05 * k
        R = P.M.so3_exp([0.0, 0.0, 0.05 * np.sin(0.2 * k)])
        gt.append((R, np.array([x, 0.0, P.stairs(x + 0.2) + 0.3])))
    scans, kinds = zip(*[P.make_scan(rng, R, t, 8000) for R, t in gt])
    res = PL.run_odometry(scans, kinds, [0.1 * k for k in range(12)], gt[0][0], gt[0][1],
                          T.Rect((-1.0, -3.0), (12.0, 3.0)),
                          lever_arms=np.array([[0.2, 0.15, -0.25], [0.2, -0.15, -0.25]]),
                          wheel_radius=0.05, config=PL.RunConfig(use_manifold=manifold))
    err = np.array([np.linalg.norm(a[1] - b[1]) for a, b in zip(res.trajectory, gt)])
    assert not any(f.held for f in res.frames)
    assert err.max() < (0.05 if not manifold else 0.10)
    assert res.terrain.num_centers() > 500
    assert all(f.terrain is not None for f in res.frames if f.inserted)
