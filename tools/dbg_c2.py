import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import numpy as np
from pipeline_c2 import make_scan, stairs
from paper_2509_26222_b200 import match as M
rng = np.random.default_rng(11)
gm = M.LocalMap(0.1, 20)
R = M.so3_exp([0, 0, 0.0]); t = np.array([0.2, 0.0, 0.3])
P, K = make_scan(rng, R, t)
print("kinds", np.bincount(K))
gm.insert(P, K, None, R, t)
print("map edge/planar", len(gm.points(0)[0]), len(gm.points(1)[0]))
R2 = M.so3_exp([0, 0, 0.01]); t2 = np.array([0.25, 0.01, 0.3])
P2, K2 = make_scan(rng, R2, t2)
c = M.build_correspondences(P2, K2, R2, t2, gm)
print("corr", len(c), "kinds", np.bincount(c.kind, minlength=2))
ne = M.feature_normal_eq(gm, R2, t2)
print("diag A", np.diag(ne.A))
print(np.linalg.eigvalsh(ne.A))
import ctypes as C
from paper_2509_26222_b200 import _abi
from paper_2509_26222_b200.terrain import Context
lam = C.c_double()
c = M._ne29(ne)
print("A[0..5]", list(c.A)[:6])
_abi.check(_abi.load().tlg_ne_min_eigenvalue(Context.default().handle, C.byref(c), C.byref(lam)))
print("device min eig", lam.value)
