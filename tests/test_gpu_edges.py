"""Edge cases of the lattice sweep and the manifold-row reduction against the
CPU oracle: queries exactly on / one ulp around the reference's hash-cell
boundaries (the 3x3 cell window is part of the reference's membership rule,
grid_index.hpp:32-48), a geometry that is not compiled in (runtime pair
classes), parameters where the separable exp recurrence is disabled, row
counts that are not multiples of a warp, empty scans and non-finite lever
arms."""
import numpy as np
import pytest

import oracle as orc
from helpers import assert_values_close, scales, so3_exp, uniform_xy
from paper_2509_26222_b200 import kinematics as kin
from paper_2509_26222_b200 import terrain as T

pytestmark = pytest.mark.gpu


def _lattice_model(sigma=0.04, sigma_eps=0.1, mesh=0.07, side=1.05, seed=61):
    k = T.KernelParams(sigma=sigma, sigma_eps=sigma_eps)
    k.finalize()
    roi = T.Rect((0.0, 0.0), (side, side))
    n = int(round(side / mesh))
    ii, jj = np.meshgrid(np.arange(n + 1), np.arange(n + 1), indexing="ij")
    nodes = np.stack([0.0 + ii.ravel() * mesh, 0.0 + jj.ravel() * mesh], 1)
    nodes = nodes[(nodes[:, 0] <= side) & (nodes[:, 1] <= side)]
    cs = T.CenterSet(nodes, mesh, 0.12, 3, roi)
    g, o = T.TerrainModel(k, cs), orc.Model(k, cs)
    w = np.cos(np.arange(len(nodes)) * 0.53 + seed)
    g.set_weights(w)
    o.set_weights(w)
    return k, cs, g, o


def _sweep(g):
    import ctypes as C
    from paper_2509_26222_b200 import _abi
    kind, rec = C.c_int(), C.c_int()
    _abi.check(_abi.load().tlg_model_sweep(g.handle, C.byref(kind), C.byref(rec)))
    return kind.value, rec.value


def _check_predict(k, g, o, q):
    z, s, gx, gy = g.predict(q)
    zr, sr, gxr, gyr = o.predict(q)
    assert np.array_equal(s, sr)
    hs, gs = scales(o, q, k.sigma)
    assert_values_close(z, zr, hs, what="height")
    assert_values_close(gx, gxr, gs, what="gx")
    assert_values_close(gy, gyr, gs, what="gy")


@pytest.mark.parametrize("exact", [False, True])
def test_queries_on_hash_cell_boundaries(gpu_ctx, exact):
    k, cs, g, o = _lattice_model()
    # compiled paper geometry; by default without the per-pair cutoff test on
    # boundary pairs (kappa_sigma(rho) = 6.8e-15), exact on request
    assert _sweep(g) == (200, 1)
    if exact:
        g.set_exact_cutoff(True)
        assert _sweep(g) == (100, 1)
    cell = k.cutoff_radius  # GridIndex2 cell = min(cutoff, 1e6)
    edges = np.arange(-1, int(1.05 / cell) + 2) * cell
    vals = np.concatenate([edges, np.nextafter(edges, -np.inf), np.nextafter(edges, np.inf)])
    rng = np.random.default_rng(5)
    q = np.stack([rng.choice(vals, 6000), rng.uniform(-0.1, 1.15, 6000)], 1)
    q = np.concatenate([q, q[:, ::-1], np.stack([rng.choice(vals, 3000), rng.choice(vals, 3000)], 1)])
    _check_predict(k, g, o, q)


def test_runtime_geometry_not_compiled(gpu_ctx):
    # mesh 0.05 -> cutoff / res = 6.46 lattice units: runtime pair classes
    k, cs, g, o = _lattice_model(mesh=0.05, side=1.0)
    kind, rec = _sweep(g)
    assert 4 <= kind <= 14 and rec == 1
    q = uniform_xy(orc.Rng(71), 4000, -0.2, 1.2)
    _check_predict(k, g, o, q)


def test_exp_recurrence_disabled(gpu_ctx):
    # sigma << sigma~ (cutoff 3 sigma~ spans ~30 sigma): the exponent range over
    # the window is too wide for the two-multiply recurrence -> one exp per node
    k, cs, g, o = _lattice_model(sigma=0.01, sigma_eps=0.1)
    kind, rec = _sweep(g)
    assert 4 <= kind <= 14 and rec == 0
    q = uniform_xy(orc.Rng(72), 3000, -0.05, 1.1)
    _check_predict(k, g, o, q)


@pytest.mark.parametrize("n", [1, 31, 33, 257, 4099])
def test_manifold_rows_ragged_sizes(gpu_ctx, n):
    k, cs, g, o = _lattice_model(seed=n)
    R = so3_exp([0.01, -0.02, 0.3])
    t = np.array([0.05, 0.02, 0.1])
    pts = np.concatenate([uniform_xy(orc.Rng(n), n, -0.05, 1.1), np.full((n, 1), 0.03)], 1)
    h = (pts - t) @ R
    rows, ne = kin.manifold_rows(g, R, t, h, 0.0, 1.0, 0.05, want=("r", "J", "valid"))
    ref, ne_ref = o.manifold_rows(R, t, h, 0.0, 1.0, 0.05)
    assert np.array_equal(rows["valid"], ref["valid"])
    A = ne.A[np.triu_indices(6)]
    scale = max(np.abs(ne_ref[:21]).max(), 1e-300)
    np.testing.assert_allclose(A, ne_ref[:21], rtol=1e-9, atol=1e-9 * scale)
    assert ne.valid == int(ne_ref[28])
    sc = kin.Scan(g, R, t, h)
    srows, sne = sc.manifold_rows(R, t, 0.0, 1.0, 0.05)
    perm = sc.permutation()
    assert np.array_equal(srows["valid"], rows["valid"][perm])
    np.testing.assert_allclose(sne.A, ne.A, rtol=1e-12, atol=1e-12 * scale)


def test_manifold_rows_empty_and_nonfinite(gpu_ctx):
    k, cs, g, o = _lattice_model()
    R = np.eye(3)
    t = np.zeros(3)
    rows, ne = kin.manifold_rows(g, R, t, np.zeros((0, 3)), 0.0, 1.0, 0.05)
    assert ne.valid == 0 and ne.cost == 0.0 and np.all(ne.A == 0.0)
    h = np.array([[0.5, 0.5, 0.0], [np.nan, 0.2, 0.0]])
    with pytest.raises(T.DomainError):
        kin.manifold_rows(g, R, t, h, 0.0, 1.0, 0.05)
    # the model stays usable after the error
    rows, ne = kin.manifold_rows(g, R, t, h[:1], 0.0, 1.0, 0.05)
    assert ne.valid == 1


def test_manifold_rows_deterministic(gpu_ctx):
    # dynamic chunk claiming must not change the reduction order
    k, cs, g, o = _lattice_model()
    R = so3_exp([0.0, 0.0, 0.2])
    t = np.array([0.0, 0.0, 0.1])
    pts = np.concatenate([uniform_xy(orc.Rng(9), 200000, 0.0, 1.05), np.zeros((200000, 1))], 1)
    h = (pts - t) @ R
    ne0 = kin.manifold_rows(g, R, t, h, 0.0, 1.0, 0.05, want=())[1]
    for _ in range(3):
        ne1 = kin.manifold_rows(g, R, t, h, 0.0, 1.0, 0.05, want=())[1]
        assert np.array_equal(ne1.A, ne0.A) and np.array_equal(ne1.g, ne0.g)
        assert ne1.cost == ne0.cost


def test_streamed_host_batch_equals_device(gpu_ctx):
    # >= 2^20 host lever arms take the sliced H2D/compute-overlap path; the
    # chunk partials and rows must equal the single-launch device-input path
    import torch
    k, cs, g, o = _lattice_model()
    n = (1 << 20) + 12345
    rng = np.random.default_rng(8)
    h = np.ascontiguousarray(np.c_[rng.uniform(-0.05, 1.1, n), rng.uniform(-0.05, 1.1, n),
                                   np.full(n, 0.03)])
    R = so3_exp([0.01, -0.02, 0.3])
    t = np.array([0.05, 0.02, 0.1])
    hs = tuple(np.ascontiguousarray(h[:, j]) for j in range(3))
    _, ne_h = kin.manifold_rows(g, R, t, hs, 0.0, 1.0, 0.05, want=())
    hd = tuple(torch.from_numpy(a).cuda() for a in hs)
    rows_d, ne_d = kin.manifold_rows(g, R, t, hd, 0.0, 1.0, 0.05, want=("r", "valid"))
    assert np.array_equal(ne_h.A, ne_d.A) and np.array_equal(ne_h.g, ne_d.g)
    assert ne_h.cost == ne_d.cost and ne_h.valid == ne_d.valid


def test_loose_cutoff_gate_off_for_wide_kernel(gpu_ctx):
    # sigma = 0.1, sigma_eps = 0.04: same cutoff (3 sigma~ = 0.3231, the
    # compiled paper geometry) but kappa_sigma(rho) = 5e-3 -> the per-pair
    # cutoff test must stay on
    k, cs, g, o = _lattice_model(sigma=0.1, sigma_eps=0.04)
    assert _sweep(g) == (100, 1)
    q = uniform_xy(orc.Rng(73), 4000, -0.1, 1.15)
    _check_predict(k, g, o, q)


def test_loose_matches_exact_cutoff(gpu_ctx):
    # the default (no test on boundary pairs) against the exact per-pair test
    # on the same device: the difference is bounded by the gate (1e-11 of the
    # window's largest |w|)
    k, cs, g, o = _lattice_model(seed=3)
    q = uniform_xy(orc.Rng(74), 20000, -0.1, 1.15)
    z0, s0, gx0, gy0 = g.predict(q)
    g.set_exact_cutoff(True)
    z1, s1, gx1, gy1 = g.predict(q)
    assert np.array_equal(s0, s1)
    wmax = np.abs(g.weights()).max()
    assert np.abs(z0 - z1).max() <= 1e-11 * wmax
    assert np.abs(gx0 - gx1).max() * k.sigma <= 1e-11 * wmax
    assert np.abs(gy0 - gy1).max() * k.sigma <= 1e-11 * wmax
    assert np.abs(z0 - z1).max() > 0.0  # the two paths really differ


def test_loose_guard_follows_weight_changes(gpu_ctx):
    # the per-cell max-|w| table behind the loose path's guard is rebuilt
    # lazily after weight changes: evaluate, then make a few weights 1e6x
    # larger (an error bound computed from the stale table would be far too
    # small near them) and compare against the oracle again
    k, cs, g, o = _lattice_model(seed=5)
    q = uniform_xy(orc.Rng(75), 6000, -0.05, 1.1)
    _check_predict(k, g, o, q)
    w = g.weights()
    w[::37] *= 1e6
    g.set_weights(w)
    o.set_weights(w)
    _check_predict(k, g, o, q)


@pytest.mark.parametrize("allow_birth", [True, False])
def test_update_rejects_nonfinite_observation_without_state_change(gpu_ctx, allow_birth):
    # TerrainObservation::validate (center_select.cpp:9-16) runs before any
    # birth or weight change, also when its flag is read together with the
    # births pre-check
    k = T.KernelParams()
    k.finalize()
    roi = T.Rect((0.0, 0.0), (1.05, 1.05))
    g = T.TerrainModel(k, T.CenterSet(np.zeros((0, 2)), 0.07, 0.12, 3, roi))
    rng = np.random.default_rng(8)
    xy = rng.uniform(0.0, 1.05, (3000, 2))
    g.recursive_update(T.TerrainObservation(xy, np.sin(xy[:, 0])))
    g.recursive_update(T.TerrainObservation(xy[:400], np.sin(xy[:400, 0])))
    w0, n0 = g.weights().copy(), g.num_centers()
    bad = rng.uniform(0.0, 1.05, (400, 2))
    bad[17, 1] = np.nan
    with pytest.raises(T.InvalidArgument):
        g.recursive_update(T.TerrainObservation(bad, np.sin(bad[:, 0])), allow_birth)
    assert g.num_centers() == n0
    assert np.array_equal(g.weights(), w0)
