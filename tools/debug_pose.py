"""Debug helper: reference odometry (with IMU) held frames vs the GPU lm_solve
from the same predicted pose (lock-step state up to that frame)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT / "oracle"), str(ROOT), str(ROOT / "tests")]
import numpy as np
import oracle as orc
from paper_2509_26222_b200 import match as M, terrain as T
from paper_2509_26222_b200.consumers import select_ground_points
REF = orc.reference()
b = REF.SimBundle("staircase", 11, 1000, 20, 30)
o = REF.odometry(b, REF.run_config_json(use_imu=True), 0)
print("held", np.nonzero(o["held"])[0], "failed", np.nonzero(o["failed"])[0])
roi4 = b.roi(); roi = T.Rect((roi4[0], roi4[1]), (roi4[2], roi4[3]))
k = T.KernelParams(); k.finalize()
terrain = T.TerrainModel(k, T.CenterSet(np.zeros((0, 2)), 0.07, 0.12, 3, roi))
lmap = M.LocalMap(0.1, 20)
for f in range(b.num_scans()):
    P, K, L = b.scan(f)
    if f > 0:
        arms = np.stack([o["hL"][f], o["hR"][f]]) if o["has_arms"][f] else None
        use_t = arms is not None and terrain.num_centers() > 0
        Rg, tg, rep = M.lm_solve(o["R_pred"][f], o["t_pred"][f], P, K, lmap, M.SolverConfig(),
                                 terrain=terrain if use_t else None, lever_arms=arms if use_t else None,
                                 wheel_radius=b.wheel_radius())
        if o["held"][f] or rep.failed or abs(np.abs(tg - o["t"][f]).max()) > 1e-9:
            print(f, "ref:", {kk: o[kk][f] for kk in ("held", "failed", "degenerate", "outer_iterations", "accepted_steps", "correspondences", "final_cost", "min_eig")})
            print(f, "gpu:", rep)
    if o["inserted"][f]:
        lmap.insert(P, K, L, o["R"][f], o["t"][f])
        obs = select_ground_points(P, K, o["R"][f], o["t"][f], roi, 2.5, 0.12, 400)
        if len(obs.z):
            terrain.recursive_update(obs)
