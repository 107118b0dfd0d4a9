import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/oracle"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import oracle as orc
from paper_2509_26222_b200 import match as M
from test_match import _scene
gm, om = M.LocalMap(0.1, 20), orc.LocalMap(0.1, 20)
for f in range(20):
    P, K, L = _scene(100 + f, 8000)
    R = orc.so3_exp([0.0, 0.0, 0.01 * f]); t = np.array([0.02 * f, 0.0, 0.0])
    Ps = (P - t) @ R
    gm.insert(Ps, K, L, R, t); om.insert(Ps, K, L, R, t)
for k in (0, 1):
    print("map eq", k, np.array_equal(gm.points(k)[0], om.points(k)[0]))
P, K, _ = _scene(7, 8000)
R = orc.so3_exp([0.002, -0.001, 0.2]); t = np.array([0.4, -0.1, 0.0])
Ps = (P - t) @ R + np.random.default_rng(3).normal(0, 0.01, P.shape)
for trim in (5.0, 0.0):
    c = M.build_correspondences(Ps, K, R, t, gm, M.MatchConfig(trim_ratio=trim))
    o = om.build_correspondences(Ps, K, R, t, {"trim_ratio": trim})
    gs, os_ = set(c.feature.tolist()), set(o["feature"].tolist())
    print("trim", trim, len(c), len(o["kind"]), "gpu-only", sorted(gs - os_)[:5], "oracle-only", sorted(os_ - gs)[:5])
    for f in sorted(os_ ^ gs)[:3]:
        print(" feature", f, "kind", K[f], "p", Ps[f])
        if f in gs: i = list(c.feature).index(f); print("  gpu", c.params[i], c.dist[i], c.fitq[i])
        if f in os_: i = list(o["feature"]).index(f); print("  orc", o["params"][i], o["dist"][i], o["fitq"][i])
    # median check
    print(" median gpu", np.sort(c.dist)[len(c)//2] if len(c) else None)
