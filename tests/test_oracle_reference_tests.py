"""The reference's own hot-path unit tests, restated against the CPU oracle.

These pin the oracle: the reference cannot be built here, so
the oracle is checked against every closed form, brute-force count, dense
normal-equation / dense-inverse oracle and FD check the reference's tests
hold for this path. Citations are /root/reference/proj/tests/unit/*.cpp.
"""
import math

import numpy as np
import pytest

import oracle as orc
from helpers import make_field, uniform_xy
from paper_2509_26222_b200.terrain import CenterSet, KernelParams, Rect


# ---- test_kernel.cpp -----------------------------------------------------------
def test_kernel_matches_gaussian_inside_cutoff():  # test_kernel.cpp:13-28
    k = KernelParams(cutoff_radius=0.5)
    k.cutoff_radius = orc.kernel_finalize(k)
    rng = orc.Rng(7)
    for _ in range(200):
        x = (rng.uniform(-0.4, 0.4), rng.uniform(-0.4, 0.4))
        c = (rng.uniform(-0.4, 0.4), rng.uniform(-0.4, 0.4))
        d2 = (x[0] - c[0]) ** 2 + (x[1] - c[1]) ** 2
        exp_ = math.exp(-d2 / (2 * 0.04 * 0.04)) if math.sqrt(d2) <= 0.5 else 0.0
        assert orc.kernel_eval(k, x, c, 0.04) == pytest.approx(exp_, rel=1e-15, abs=0)


def test_kernel_exactly_zero_beyond_cutoff():  # :30-37
    k = KernelParams(cutoff_radius=0.5)
    k.cutoff_radius = orc.kernel_finalize(k)
    assert k.cutoff_radius == 0.5
    assert orc.kernel_eval(k, (0.0, 0.0), (0.500001, 0.0), 0.2) == 0.0
    assert orc.kernel_eval(k, (0.0, 0.0), (0.499999, 0.0), 0.2) > 0.0


def test_widened_bandwidth_and_moment_scale():  # :39-48
    k = KernelParams(sigma=0.04, sigma_eps=0.1)
    assert orc.sigma_tilde(k) == pytest.approx(math.sqrt(0.04 ** 2 + 0.1 ** 2), rel=1e-15)
    assert orc.moment_scale(k) == pytest.approx(0.04 ** 2 / (0.04 ** 2 + 0.1 ** 2), rel=1e-15)
    # SPEC.md:72 known answer s = 0.137931; kappa(|x-c| = b) = e^-1/2
    assert orc.moment_scale(k) == pytest.approx(0.137931, abs=1e-6)
    k.cutoff_radius = orc.kernel_finalize(k)
    b = orc.sigma_tilde(k)
    assert orc.kernel_eval(k, (0.0, 0.0), (b, 0.0), b) == pytest.approx(math.exp(-0.5), rel=1e-15)


def test_finalize_auto_cutoff_and_rejects():  # :50-69
    k = KernelParams()
    assert orc.kernel_finalize(k) == pytest.approx(3.0 * orc.sigma_tilde(k))
    assert orc.kernel_finalize(KernelParams(cutoff_radius=2.0)) == 2.0
    for bad in (KernelParams(sigma=0.0), KernelParams(lambda_=-1.0), KernelParams(sigma_eps=-0.1)):
        with pytest.raises(orc.OracleError) as e:
            orc.kernel_finalize(bad)
        assert e.value.status == orc.INVALID_ARGUMENT


def test_nonfinite_inputs_rejected():  # :71-77
    k = KernelParams()
    k.cutoff_radius = orc.kernel_finalize(k)
    with pytest.raises(orc.OracleError) as e:
        orc.kernel_eval(k, (math.nan, 0.0), (0.0, 0.0), 0.1)
    assert e.value.status == orc.DOMAIN_ERROR


# ---- test_center_select.cpp ------------------------------------------------------
def _support(xy, node, r):
    return int((np.hypot(xy[:, 0] - node[0], xy[:, 1] - node[1]) <= r).sum())


def test_selected_centers_satisfy_support_rule():  # test_center_select.cpp:21-36
    xy = uniform_xy(orc.Rng(11), 400, 0.0, 2.0)
    roi = Rect((0.0, 0.0), (2.0, 2.0))
    nodes = orc.supported_mesh_nodes(xy, np.zeros(400), roi, 0.1, 0.12, 3, throw_empty=True)
    assert len(nodes)
    for c in nodes:
        assert roi.contains(c)
        assert _support(xy, c, 0.12) >= 3


def test_no_qualifying_node_omitted():  # :38-56 (brute-force oracle)
    xy = uniform_xy(orc.Rng(12), 150, 0.0, 1.0)
    roi = Rect((0.0, 0.0), (1.0, 1.0))
    res, radius = 0.15, 0.1
    nodes = orc.supported_mesh_nodes(xy, np.zeros(150), roi, res, radius, 2, throw_empty=True)
    qualifying = 0
    x = roi.min[0]
    while x <= roi.max[0] + 1e-12:
        y = roi.min[1]
        while y <= roi.max[1] + 1e-12:
            qualifying += _support(xy, (x, y), radius) >= 2
            y += res
        x += res
    assert len(nodes) == qualifying


def test_centers_on_lattice():  # :58-73
    xy = np.array([[0.5 + 0.01 * i, 0.5] for i in range(20)])
    nodes = orc.supported_mesh_nodes(xy, np.zeros(20), Rect((0.0, 0.0), (1.0, 1.0)), 0.2, 0.15, 3,
                                     throw_empty=True)
    f = nodes / 0.2
    assert np.all(np.abs(f - np.round(f)) < 1e-9)


def test_unsupported_region_raises():  # :75-82
    xy, z = np.array([[10.0, 10.0]]), np.zeros(1)
    roi = Rect((0.0, 0.0), (1.0, 1.0))
    with pytest.raises(orc.OracleError) as e:
        orc.supported_mesh_nodes(xy, z, roi, 0.1, 0.1, 3, throw_empty=True)
    assert e.value.status == orc.NO_SUPPORTED_CENTERS
    assert len(orc.supported_mesh_nodes(xy, z, roi, 0.1, 0.1, 3)) == 0


def test_observation_validation():  # :84-93
    roi = Rect((0.0, 0.0), (1.0, 1.0))
    for xy, z in ((np.zeros((0, 2)), np.zeros(0)), (np.zeros((1, 2)), np.zeros(0)),
                  (np.zeros((1, 2)), np.array([np.inf]))):
        with pytest.raises(orc.OracleError) as e:
            orc.supported_mesh_nodes(xy, z, roi, 0.1, 0.1, 1)
        assert e.value.status == orc.INVALID_ARGUMENT
    orc.supported_mesh_nodes(np.zeros((1, 2)), np.ones(1), roi, 0.1, 0.1, 1)


def test_grid_index_matches_brute_force():  # test_io_pipeline.cpp:43-59
    rng = orc.Rng(72)
    pts = uniform_xy(rng, 400, 0.0, 5.0)
    g = orc.Grid(0.3, pts)
    for trial in range(40):
        q = (rng.uniform(0.0, 5.0), rng.uniform(0.0, 5.0))
        r = 0.05 + 0.1 * (trial % 5)
        got = g.radius_query(q, r)
        d = np.hypot(pts[:, 0] - q[0], pts[:, 1] - q[1])
        assert len(got) == int((d <= r).sum())
        assert np.all(d[got] <= r + 1e-12)
        assert np.all(np.diff(got.astype(np.int64)) > 0)  # sorted ids


# ---- test_terrain_model.cpp ------------------------------------------------------
def _dense_m(model, xy):
    n = model.num_centers()
    M = np.zeros((len(xy), n))
    for i, q in enumerate(xy):
        ids, vals = model.moment_feature(q)
        M[i, ids] = vals
    return M


def _dense_ridge(model, xy, z, lam):  # test_terrain_model.cpp:42-56
    M = _dense_m(model, xy)
    H = lam * np.eye(M.shape[1]) + M.T @ M
    return np.linalg.solve(H, M.T @ z)


def test_moment_features_formula():  # :60-77
    k, cs, obs = make_field(21)
    m = orc.Model(k, cs)
    rng = orc.Rng(22)
    st = orc.sigma_tilde(k)
    for _ in range(50):
        x = (rng.uniform(0.0, 1.0), rng.uniform(0.0, 1.0))
        ids, vals = m.moment_feature(x)
        for j, v in zip(ids, vals):
            d2 = (x[0] - cs.centers[j][0]) ** 2 + (x[1] - cs.centers[j][1]) ** 2
            assert v == pytest.approx(orc.moment_scale(k) * math.exp(-d2 / (2 * st * st)), rel=1e-14)
            assert math.sqrt(d2) <= k.cutoff_radius + 1e-12


def test_predict_height_is_plain_expansion():  # :79-100
    k, cs, obs = make_field(23)
    m = orc.fit_batch_ridge(k, cs, obs.xy, obs.z)
    rng = orc.Rng(24)
    w = m.weights()
    c = np.asarray(cs.centers)
    q = np.array([(rng.uniform(0.1, 0.9), rng.uniform(0.1, 0.9)) for _ in range(50)])
    z, s, _, _ = m.predict(q)
    for i, x in enumerate(q):
        d = np.hypot(c[:, 0] - x[0], c[:, 1] - x[1])
        sel = d <= k.cutoff_radius
        manual = (w[sel] * np.exp(-d[sel] ** 2 / (2 * k.sigma ** 2))).sum()
        assert s[i] == 1
        assert z[i] == pytest.approx(manual, rel=1e-12)
    zf, sf, _, _ = m.predict(np.array([[50.0, 50.0]]))
    assert sf[0] == 0 and zf[0] == 0.0


def test_batch_fit_matches_dense_oracle():  # :102-107
    k, cs, obs = make_field(25, 200, 0.15, 10.0)
    m = orc.fit_batch_ridge(k, cs, obs.xy, obs.z)
    ref = _dense_ridge(m, obs.xy, obs.z, k.lambda_)
    assert np.linalg.norm(m.weights() - ref) / np.linalg.norm(ref) < 1e-10


def test_recursive_reproduces_batch():  # :109-126
    k, cs, obs = make_field(26, 400, 0.15, 10.0)
    m = orc.Model(k, cs)
    splits, chunk = 8, len(obs.xy) // 8
    for s in range(splits):
        b = s * chunk
        e = len(obs.xy) if s == splits - 1 else b + chunk
        assert not m.recursive_update(obs.xy[b:e], obs.z[b:e], False)["rejected"]
    batch = orc.fit_batch_ridge(k, cs, obs.xy, obs.z)
    wb = batch.weights()
    assert np.linalg.norm(m.weights() - wb) / np.linalg.norm(wb) < 1e-10


def test_block_info_inverse_tracks_dense_inverse():  # :128-148
    k, cs, obs = make_field(27, 150, 0.2, 10.0)
    m = orc.Model(k, cs)
    assert m.num_blocks() == 1
    m.recursive_update(obs.xy[:60], obs.z[:60], False)
    M = _dense_m(m, obs.xy[:60])
    expected = np.linalg.inv(k.lambda_ * np.eye(M.shape[1]) + M.T @ M)
    got = m.block_info_inverse(0)
    assert np.linalg.norm(got - expected) / np.linalg.norm(expected) < 1e-9


def test_updates_touch_only_reachable_blocks():  # :150-195
    k = KernelParams(sigma=0.08, sigma_eps=0.05)
    k.cutoff_radius = orc.kernel_finalize(k)
    xy, z = [], []
    for i in range(40):
        xy += [[0.02 * i, 0.0], [30.0 + 0.02 * i, 0.0]]
        z += [0.1, 0.5]
    xy, z = np.array(xy), np.array(z)
    roi = Rect((-1.0, -1.0), (32.0, 1.0))
    cs = CenterSet(orc.supported_mesh_nodes(xy, z, roi, 0.1, 0.15, 3, True), 0.1, 0.15, 3, roi)
    m = orc.Model(k, cs)
    assert m.num_blocks() >= 2
    before = [m.block_info_inverse(b) for b in range(m.num_blocks())]
    near = xy[:, 0] < 5.0
    m.recursive_update(xy[near], z[near], False)
    for b in range(m.num_blocks()):
        far = cs.centers[m.block_members(b)[0]][0] > 10.0
        if far:
            assert np.array_equal(m.block_info_inverse(b), before[b])
    w = m.weights()
    assert np.all(w[np.asarray(cs.centers)[:, 0] > 10.0] == 0.0)


def test_center_birth():  # :197-224
    k = KernelParams(sigma=0.08, sigma_eps=0.05)
    k.cutoff_radius = orc.kernel_finalize(k)
    first = np.array([[0.3 + 0.01 * i, 0.5] for i in range(50)])
    roi = Rect((0.0, 0.0), (3.0, 1.0))
    cs = CenterSet(orc.supported_mesh_nodes(first, np.full(50, 0.2), roi, 0.1, 0.15, 3, True),
                   0.1, 0.15, 3, roi)
    m = orc.Model(k, cs)
    m.recursive_update(first, np.full(50, 0.2))
    n0 = m.num_centers()
    second = np.array([[2.0 + 0.01 * i, 0.5] for i in range(50)])
    rep = m.recursive_update(second, np.full(50, 0.4))
    assert rep["born_centers"] > 0 and m.num_centers() > n0
    z, s, _, _ = m.predict(np.array([[2.25, 0.5]]))
    assert s[0] == 1 and z[0] == pytest.approx(0.4, rel=0.1)


def test_snapshot_round_trip(tmp_path):  # :226-241
    k, cs, obs = make_field(28)
    m = orc.fit_batch_ridge(k, cs, obs.xy, obs.z)
    p = tmp_path / "model.bin"
    m.save(p)
    l = orc.Model.load_file(p)
    assert l.num_centers() == m.num_centers()
    q = uniform_xy(orc.Rng(29), 20, 0.1, 0.9)
    np.testing.assert_allclose(l.predict(q)[0], m.predict(q)[0], rtol=1e-14)


# ---- acceptance criteria 1-2 (acceptance_main.cpp:70-150) ------------------------
def _random_field(rng, n_points, side, mesh, truncated):
    amp = orc.Normal(0.0, 0.2)
    k = KernelParams(sigma=0.08, sigma_eps=0.05, cutoff_radius=0.0 if truncated else 1e3)
    k.cutoff_radius = orc.kernel_finalize(k)
    a, b, c = amp.draw(rng), amp.draw(rng), amp.draw(rng)
    xy = uniform_xy(rng, n_points, 0.0, side)
    z = a * np.sin(3 * xy[:, 0]) + b * np.cos(2 * xy[:, 1]) + c * xy[:, 0] * xy[:, 1]
    roi = Rect((0.0, 0.0), (side, side))
    cs = CenterSet(orc.supported_mesh_nodes(xy, z, roi, mesh, 1.6 * mesh, 3, True), mesh,
                   1.6 * mesh, 3, roi)
    return k, cs, xy, z


def test_acceptance_1_batch_recursive_equivalence():
    rng = orc.Rng(101)
    worst = 0.0
    for _ in range(2):
        k, cs, xy, z = _random_field(rng, 2000, 1.2, 0.1, False)
        assert len(cs.centers) <= 200
        rec = orc.Model(k, cs)
        chunk = len(xy) // 10
        for s in range(10):
            b = s * chunk
            e = len(xy) if s == 9 else b + chunk
            rec.recursive_update(xy[b:e], z[b:e], False)
        wb = orc.fit_batch_ridge(k, cs, xy, z).weights()
        worst = max(worst, np.linalg.norm(rec.weights() - wb) / np.linalg.norm(wb))
    assert worst < 1e-8


def test_acceptance_2_woodbury_block_update():
    rng = orc.Rng(102)
    worst = 0.0
    for _ in range(30):
        k = KernelParams(sigma=0.08, sigma_eps=0.05, cutoff_radius=1e3)
        k.cutoff_radius = orc.kernel_finalize(k)
        n = rng.uniform_int(5, 30)
        c = np.array([(rng.uniform(0.0, 0.5), rng.uniform(0.0, 0.5)) for _ in range(n)])
        cs = CenterSet(c, 0.07, 0.07, 3, Rect((0.0, 0.0), (0.5, 0.5)))
        m = orc.Model(k, cs)
        prior = np.array([(rng.uniform(0.0, 0.5), rng.uniform(0.0, 0.5)) for _ in range(20)])
        pz = np.array([rng.uniform(0.0, 0.5) for _ in range(20)])
        m.recursive_update(prior, pz, False)
        h_prev = np.linalg.inv(m.block_info_inverse(0))
        x = np.array([[rng.uniform(0.0, 0.5), rng.uniform(0.0, 0.5)]])
        mv = _dense_m(m, x)[0]
        m.recursive_update(x, np.array([rng.uniform(0.0, 0.5)]), False)
        expected = np.linalg.inv(h_prev + np.outer(mv, mv))
        got = m.block_info_inverse(0)
        worst = max(worst, np.linalg.norm(got - expected) / np.linalg.norm(expected))
    assert worst < 1e-8


def test_acceptance_3_gradient_fd():  # acceptance_main.cpp:154-185
    rng = orc.Rng(103)
    k, cs, xy, z = _random_field(rng, 400, 1.0, 0.1, True)
    m = orc.fit_batch_ridge(k, cs, xy, z)
    h = 1e-6
    worst, checked = 0.0, 0
    while checked < 40:
        q = np.array([[rng.uniform(0.15, 0.85), rng.uniform(0.15, 0.85)]])
        zq, s, gx, gy = m.predict(q)
        if not s[0] or math.hypot(gx[0], gy[0]) < 1e-3:
            continue
        pts = q + np.array([[h, 0], [-h, 0], [0, h], [0, -h]])
        zz = m.predict(pts)[0]
        fd = np.array([(zz[0] - zz[1]) / (2 * h), (zz[2] - zz[3]) / (2 * h)])
        worst = max(worst, np.linalg.norm(fd - [gx[0], gy[0]]) / np.linalg.norm(fd))
        checked += 1
    assert worst < 1e-5


# ---- test_kinematics.cpp: manifold residual / Jacobian -----------------------------
def _flat_terrain(height):  # test_kinematics.cpp:40-56
    k = KernelParams(sigma=0.08, sigma_eps=0.02)
    k.cutoff_radius = orc.kernel_finalize(k)
    rng = orc.Rng(31)
    xy = uniform_xy(rng, 900, -1.5, 1.5)
    z = np.full(900, height)
    roi = Rect((-1.5, -1.5), (1.5, 1.5))
    cs = CenterSet(orc.supported_mesh_nodes(xy, z, roi, 0.1, 0.12, 3, True), 0.1, 0.12, 3, roi)
    return orc.fit_batch_ridge(k, cs, xy, z)


def test_manifold_residual_is_contact_height():  # :85-100
    m = _flat_terrain(0.2)
    R = np.eye(3)
    t = np.array([0.0, 0.0, 0.9])
    hlev = np.array([[0.05, 0.15, -0.55]])
    rows, ne = m.manifold_rows(R, t, hlev, 0.08, 1.0, 0.0)
    wc = R @ hlev[0] + t
    f = m.predict(wc[None, :2])[0][0]
    assert rows["valid"][0] == 1
    assert rows["raw"][0] == pytest.approx(wc[2] - 0.08 - f, rel=1e-12)


def test_unsupported_terrain_invalidates():  # :102-111
    m = _flat_terrain(0.0)
    rows, ne = m.manifold_rows(np.eye(3), np.array([100.0, 0.0, 0.6]),
                               np.array([[0.0, 0.15, -0.58]]), 0.08, 1.0, 0.05)
    assert rows["valid"][0] == 0 and rows["r"][0] == 0.0 and np.all(rows["J"] == 0.0)
    assert ne[28] == 0.0


def test_manifold_jacobian_central_difference():  # :113-144
    m = _flat_terrain(0.1)
    rng = orc.Rng(32)
    checked = 0
    for _ in range(30):
        u = lambda: rng.uniform(-0.3, 0.3)  # noqa: E731
        hlev = np.array([[0.1 * u(), 0.15 + 0.1 * u(), -0.5 + 0.1 * u()]])
        R = orc.so3_exp([0.3 * u(), 0.3 * u(), u()])
        t = np.array([u(), u(), 0.7 + 0.1 * u()])
        base, _ = m.manifold_rows(R, t, hlev, 0.08, 1.0, 0.0)
        if not base["valid"][0]:
            continue
        J = base["J"][0]
        h = 1e-6
        for d in range(6):
            def val(eps):
                delta = np.zeros(3)
                delta[d % 3] = eps
                if d < 3:
                    Rp, tp = R @ orc.so3_exp(delta), t
                else:
                    Rp, tp = R, t + delta
                return m.manifold_rows(Rp, tp, hlev, 0.08, 1.0, 0.0)[0]["raw"][0]
            fd = (val(h) - val(-h)) / (2 * h)
            assert abs(fd - J[d]) < 1e-4 * max(1.0, abs(fd))
        checked += 1
    assert checked > 10


def test_zero_lambda_manifold_is_inert():  # test_matcher.cpp:150-184 (lambda_M = 0 rows vanish)
    m = _flat_terrain(0.1)
    rows, ne = m.manifold_rows(np.eye(3), np.zeros(3), np.array([[0.1, 0.1, 0.05]] * 5), 0.0, 0.0,
                               0.05)
    assert np.all(rows["r"] == 0.0) and np.all(rows["J"] == 0.0)
    assert np.all(ne[:28] == 0.0)
