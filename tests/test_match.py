"""Feature correspondences: the device LocalMap, kNN line /
plane association and the total_cost feature rows vs the oracle restatement
of local_map.cpp / kdtree.hpp / scan_matcher.cpp. Map contents, kNN ids,
correspondence sets, labels and (with the shared Jacobi eigen sweeps)
parameters are bit-exact; the normal equations agree to 1e-12 (different
summation order)."""
import numpy as np
import pytest

import oracle as orc
from helpers import so3_exp
from paper_2509_26222_b200 import match as M


def _scene(seed, n=3000):
    """Ground plane, two walls, vertical edges (poles), with labels."""
    rng = np.random.default_rng(seed)
    g = np.c_[rng.uniform(-5, 5, n), rng.uniform(-5, 5, n), rng.normal(0, 0.004, n)]
    w1 = np.c_[np.full(n // 2, 3.0) + rng.normal(0, 0.004, n // 2), rng.uniform(-5, 5, n // 2),
               rng.uniform(0, 2.5, n // 2)]
    w2 = np.c_[rng.uniform(-5, 3, n // 2), np.full(n // 2, 4.0) + rng.normal(0, 0.004, n // 2),
               rng.uniform(0, 2.5, n // 2)]
    poles = []
    for k, (x, y) in enumerate([(1.0, 1.0), (-2.0, 0.5), (0.5, -3.0)]):
        m = 300
        poles.append(np.c_[np.full(m, x), np.full(m, y), rng.uniform(0, 2.5, m)] +
                     rng.normal(0, 0.002, (m, 3)))
    e = np.concatenate(poles)
    P = np.concatenate([g, w1, w2, e])
    K = np.concatenate([np.full(len(g), 2), np.ones(len(w1) + len(w2)), np.zeros(len(e))])
    L = np.concatenate([np.zeros(len(g)), np.full(len(w1), 1), np.full(len(w2), 2),
                        np.repeat([3, 4, 5], 300)])
    perm = rng.permutation(len(P))
    return P[perm], K[perm].astype(np.uint8), L[perm].astype(np.int32)


def _maps(seed, frames=3, gpu=True):
    gm, om = (M.LocalMap(0.1, 20) if gpu else None), orc.LocalMap(0.1, 20)
    for f in range(frames):
        P, K, L = _scene(seed + f)
        R = so3_exp([0.0, 0.0, 0.02 * f])
        t = np.array([0.05 * f, -0.03 * f, 0.0])
        Ps = (P - t) @ R  # sensor frame so that R Ps + t = P
        if gpu:
            gm.insert(Ps, K, L, R, t)
        om.insert(Ps, K, L, R, t)
    return gm, om


def test_oracle_knn_and_fits_sane():
    _, om = _maps(1, frames=1, gpu=False)
    pts, _ = om.points(1)
    q = pts[10] + 0.01
    ids = om.knn(1, q, 8, 1.0)
    d = np.sum((pts[ids] - q) ** 2, 1)
    assert len(ids) == 8 and np.all(np.diff(d) >= 0)
    brute = np.argsort(np.sum((pts - q) ** 2, 1), kind="stable")[:8]
    assert set(ids) == set(brute)
    # the restated kd-tree (reference algorithm) equals the exhaustive search
    rng = np.random.default_rng(3)
    for kind in (0, 1):
        p, _ = om.points(kind)
        for _ in range(200):
            qq = p[rng.integers(len(p))] + rng.normal(0, 0.05, 3)
            for k in (5, 8):
                assert np.array_equal(om.knn(kind, qq, k, 0.3, tree=True),
                                      om.knn(kind, qq, k, 0.3, tree=False))


@pytest.mark.gpu
def test_map_insert_bit_exact(gpu_ctx):
    gm, om = _maps(3)
    for kind in (0, 1):
        gp, gl = gm.points(kind)
        op, ol = om.points(kind)
        assert gp.shape == op.shape
        assert np.array_equal(gp.view(np.uint64), op.view(np.uint64))
        assert np.array_equal(gl, ol)


@pytest.mark.gpu
@pytest.mark.parametrize("trim", [5.0, 0.0])
def test_correspondences_parity(gpu_ctx, trim):
    gm, om = _maps(5)
    P, K, _ = _scene(99, 2000)
    R = so3_exp([0.003, -0.002, 0.04])
    t = np.array([0.08, -0.05, 0.01])
    Ps = (P - t) @ R + np.random.default_rng(1).normal(0, 0.01, P.shape)
    cfg = M.MatchConfig(trim_ratio=trim)
    g = M.build_correspondences(Ps, K, R, t, gm, cfg)
    o = om.build_correspondences(Ps, K, R, t, {"trim_ratio": trim})
    assert len(g) == len(o["kind"]) and len(g) > 100
    assert np.array_equal(g.feature, o["feature"])
    assert np.array_equal(g.kind, o["kind"])
    assert np.array_equal(g.label, o["label"])
    assert np.array_equal(g.params.view(np.uint64), o["params"].view(np.uint64))
    assert np.array_equal(g.weight, o["weight"]) and np.array_equal(g.dist, o["dist"])
    ne = M.feature_normal_eq(gm, R, t)
    ne_ref = orc.feature_normal_eq(o, Ps, R, t)
    A = ne.A[np.triu_indices(6)]
    np.testing.assert_allclose(A, ne_ref[:21], rtol=1e-12, atol=1e-12 * np.abs(ne_ref[:21]).max())
    np.testing.assert_allclose(ne.g, ne_ref[21:27], rtol=1e-12,
                               atol=1e-12 * np.abs(ne_ref[21:27]).max())
    assert abs(ne.cost - ne_ref[27]) <= 1e-12 * ne_ref[27]
    assert ne.valid == int(ne_ref[28])


@pytest.mark.gpu
def test_correspondences_empty_map_and_window(gpu_ctx):
    gm = M.LocalMap(0.1, 2)
    g = M.build_correspondences(np.zeros((5, 3)), np.zeros(5, dtype=np.uint8), np.eye(3),
                                np.zeros(3), gm)
    assert len(g) == 0
    # the window keeps the last two frames only (local_map.cpp:44)
    om = orc.LocalMap(0.1, 2)
    for f in range(4):
        P, K, L = _scene(20 + f, 600)
        gm.insert(P, K, L, np.eye(3), np.zeros(3))
        om.insert(P, K, L, np.eye(3), np.zeros(3))
    for kind in (0, 1):
        assert np.array_equal(gm.points(kind)[0], om.points(kind)[0])


@pytest.mark.gpu
def test_lm_step_matches_oracle(gpu_ctx):
    gm, om = _maps(7, frames=2)
    P, K, _ = _scene(70, 1500)
    R = so3_exp([0.002, 0.001, 0.03])
    t = np.array([0.05, 0.02, 0.0])
    Ps = (P - t) @ R + np.random.default_rng(2).normal(0, 0.01, P.shape)
    M.build_correspondences(Ps, K, R, t, gm)
    ne = M.feature_normal_eq(gm, R, t)
    for mu in (1e-4, 1e-2, 1.0):
        d = M.lm_step(ne, mu)
        ne29 = np.concatenate([ne.A[np.triu_indices(6)], ne.g, [ne.cost, ne.valid]])
        dref, ok = orc.lm_step(ne29, mu)
        assert ok
        np.testing.assert_array_equal(d, dref)


@pytest.mark.gpu
def test_map_voxel_key_all_ones(gpu_ctx):
    # points with x, y, z in [-voxel, 0): every 21-bit voxel field is 0x1fffff,
    # i.e. an all-ones key — must still be kept (regression)
    P = np.array([[-0.05, -0.05, -0.05], [-0.02, -0.07, -0.01], [0.3, 0.3, 0.3]])
    K = np.array([1, 1, 1], dtype=np.uint8)
    gm, om = M.LocalMap(0.1, 20), orc.LocalMap(0.1, 20)
    gm.insert(P, K, np.zeros(3), np.eye(3), np.zeros(3))
    om.insert(P, K, np.zeros(3), np.eye(3), np.zeros(3))
    assert np.array_equal(gm.points(1)[0], om.points(1)[0])
    assert len(gm.points(1)[0]) == 2


@pytest.mark.gpu
def test_lm_solve_recovers_pose(gpu_ctx):
    # map built at known poses; a new scan seen from a displaced pose is
    # registered from a perturbed guess (scan_matcher.cpp:257-358)
    gm = M.LocalMap(0.1, 20)
    for f in range(4):
        P, K, L = _scene(200 + f, 3000)
        gm.insert(P, K, L, np.eye(3), np.zeros(3))
    P, K, _ = _scene(300, 3000)
    R_true = so3_exp([0.01, -0.005, 0.15])
    t_true = np.array([0.3, -0.2, 0.02])
    Ps = (P - t_true) @ R_true + np.random.default_rng(5).normal(0, 0.003, P.shape)
    R0 = R_true @ so3_exp([0.004, -0.003, 0.03])
    t0 = t_true + np.array([0.05, -0.04, 0.01])
    R, t, rep = M.lm_solve(R0, t0, Ps, K, gm)
    assert not rep.failed and rep.accepted_steps > 0
    assert np.linalg.norm(t - t_true) < 5e-3
    ang = np.arccos(np.clip((np.trace(R.T @ R_true) - 1) / 2, -1, 1))
    assert ang < 1e-3
    assert rep.cost_trace[-1] < rep.cost_trace[0]


@pytest.mark.gpu
def test_min_eigenvalue_probe(gpu_ctx):
    # the degeneracy probe of lm_solve against numpy on random SPD 6x6 matrices
    import ctypes as C
    from paper_2509_26222_b200 import _abi
    from paper_2509_26222_b200.kinematics import NormalEq
    from paper_2509_26222_b200.terrain import Context
    rng = np.random.default_rng(4)
    for _ in range(20):
        G = rng.standard_normal((6, 6)) * rng.uniform(0.1, 100, 6)
        A = G @ G.T
        lam = C.c_double()
        c = M._ne29(NormalEq(A, np.zeros(6), 0.0, 0))
        _abi.check(_abi.load().tlg_ne_min_eigenvalue(Context.default().handle, C.byref(c),
                                                     C.byref(lam)))
        ref = np.linalg.eigvalsh(A)[0]
        assert abs(lam.value - ref) <= 1e-9 * np.abs(np.linalg.eigvalsh(A)).max()
