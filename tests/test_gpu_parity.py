"""GPU parity: the sm_100a path through the C-ABI vs the CPU oracle on the
same seeded inputs. Indexing (node lists, neighbour ids, supported flags,
block ids) must be bit-exact; heights/gradients/Jacobians within 1e-9 of
max(|ref|, sum|w kappa|); weights / info_inv within 1e-8 relative (norm)."""
import os

import numpy as np
import pytest

import oracle as orc
from helpers import (assert_manifold_rows_close, assert_values_close, c1_inputs, make_field,
                     manifold_row_scales, rel_norm, scales, so3_exp, uniform_xy)
from paper_2509_26222_b200 import kinematics as kin
from paper_2509_26222_b200 import terrain as T

pytestmark = pytest.mark.gpu

ROI1 = T.Rect((0.0, 0.0), (1.05, 1.05))


def _models(kernel, centers):
    return T.TerrainModel(kernel, centers), orc.Model(kernel, centers)


def _fitted_pair(seed=23, n_points=300, mesh=0.12, cutoff=0.0):
    k, cs, obs = make_field(seed, n_points, mesh, cutoff)
    g = T.fit_batch_ridge(k, cs, obs)
    o = orc.fit_batch_ridge(k, cs, obs.xy, obs.z)
    return k, cs, obs, g, o


# ---- K2 select ----------------------------------------------------------------
@pytest.mark.parametrize("seed,n,res,ra,count", [(11, 400, 0.1, 0.12, 3), (12, 150, 0.15, 0.1, 2),
                                                  (2509, 20000, 0.07, 0.12, 3)])
def test_select_centers_bit_exact(gpu_ctx, seed, n, res, ra, count):
    rng = orc.Rng(seed)
    xy = uniform_xy(rng, n, 0.0, 2.0)
    z = np.zeros(n)
    roi = T.Rect((0.0, 0.0), (2.0, 2.0))
    got = T.supported_mesh_nodes(T.TerrainObservation(xy, z), roi, res, ra, count)
    ref = orc.supported_mesh_nodes(xy, z, roi, res, ra, count)
    assert got.shape == ref.shape
    assert np.array_equal(got.view(np.uint64), ref.view(np.uint64))  # bits + order


def test_select_centers_errors(gpu_ctx):
    roi = T.Rect((0.0, 0.0), (1.0, 1.0))
    far = T.TerrainObservation(np.array([[10.0, 10.0]]), np.array([0.0]))
    with pytest.raises(T.NoSupportedCenters):
        T.select_centers(far, roi, 0.1, 0.1, 3)
    assert len(T.supported_mesh_nodes(far, roi, 0.1, 0.1, 3)) == 0
    with pytest.raises(T.InvalidArgument):
        T.select_centers(T.TerrainObservation(np.zeros((0, 2)), np.zeros(0)), roi, 0.1, 0.1, 3)
    with pytest.raises(T.InvalidArgument):
        T.select_centers(T.TerrainObservation(np.zeros((1, 2)), np.array([np.inf])), roi, 0.1, 0.1, 3)
    with pytest.raises(T.InvalidArgument):
        T.select_centers(far, roi, 0.0, 0.1, 3)


# ---- K3 eval --------------------------------------------------------------------
def test_eval_parity_fitted(gpu_ctx):
    k, cs, obs, g, o = _fitted_pair()
    rng = orc.Rng(24)
    q = uniform_xy(rng, 4000, -0.2, 1.2)
    z, s, gx, gy = g.predict(q)
    zr, sr, gxr, gyr = o.predict(q)
    assert np.array_equal(s, sr)
    hs, gs = scales(o, q, k.sigma)
    assert_values_close(z, zr, hs, what="height")
    assert_values_close(gx, gxr, gs, what="grad x")
    assert_values_close(gy, gyr, gs, what="grad y")
    assert np.all(z[s == 0] == 0.0)


def test_eval_c1_parity(gpu_ctx):
    xy, z = c1_inputs(20000)
    k = T.KernelParams()
    k.finalize()
    cs = T.select_centers(T.TerrainObservation(xy, z), ROI1, 0.07, 0.12, 3)
    ref_nodes = orc.supported_mesh_nodes(xy, z, ROI1, 0.07, 0.12, 3)
    assert np.array_equal(cs.centers, ref_nodes)
    assert len(cs.centers) == 256
    g, o = _models(k, cs)
    w = np.sin(np.arange(256) * 0.37)
    g.set_weights(w)
    o.set_weights(w)
    z1, s1, gx1, gy1 = g.predict(xy)
    z2, s2, gx2, gy2 = o.predict(xy)
    assert np.array_equal(s1, s2)
    hs, gs = scales(o, xy[:3000], k.sigma)
    assert_values_close(z1[:3000], z2[:3000], hs, what="height")
    assert_values_close(gx1[:3000], gx2[:3000], gs, what="gx")
    assert_values_close(gy1[:3000], gy2[:3000], gs, what="gy")


def test_eval_device_tensors(gpu_ctx):
    import torch
    k, cs, obs, g, o = _fitted_pair(seed=28)
    q = uniform_xy(orc.Rng(5), 1000, 0.0, 1.0)
    zd, sd, gxd, gyd = g.predict(torch.from_numpy(q).cuda())
    zh, sh, _, _ = g.predict(q)
    assert np.array_equal(zd.cpu().numpy(), zh)
    assert np.array_equal(sd.cpu().numpy(), sh)


def test_eval_nonfinite_is_domain_error(gpu_ctx):
    k, cs, obs, g, o = _fitted_pair()
    with pytest.raises(T.DomainError):
        g.predict(np.array([[np.nan, 0.5]]))


def test_moment_features_ids_bit_exact(gpu_ctx):
    k, cs, obs, g, o = _fitted_pair(seed=21)
    q = uniform_xy(orc.Rng(22), 200, 0.0, 1.0)
    rp, ids, vals = g.moment_features(q)
    for i in range(len(q)):
        rid, rval = o.moment_feature(q[i])
        gid = ids[rp[i]:rp[i + 1]]
        gval = vals[rp[i]:rp[i + 1]]
        assert np.array_equal(gid, rid)
        np.testing.assert_allclose(gval, rval, rtol=1e-14, atol=0)


# ---- K4 manifold rows ---------------------------------------------------------
def test_manifold_rows_parity(gpu_ctx):
    k, cs, obs, g, o = _fitted_pair(seed=31, n_points=900)
    R = so3_exp([0.02, -0.015, 0.04])
    t = np.array([0.1, -0.05, 0.08])
    pts = np.concatenate([uniform_xy(orc.Rng(7), 5000, -0.1, 1.1),
                          np.full((5000, 1), 0.05)], 1)
    h = (pts - t) @ R  # R^T (p - t)
    rows, ne = kin.manifold_rows(g, R, t, h, 0.0, 1.0, 0.05, want=("r", "J", "valid", "raw"))
    ref, ne_ref = o.manifold_rows(R, t, h, 0.0, 1.0, 0.05)
    assert np.array_equal(rows["valid"], ref["valid"])
    J = rows["J"].reshape(6, -1).T
    # SURVEY §8d scale, no additive floor: r and J within 1e-9 of
    # max(|ref|, s sum|w kappa| (...)) per row
    sc = manifold_row_scales(o, R, t, h, ref["J"])
    assert_manifold_rows_close(rows["r"], J, ref["r"], ref["J"], sc, rtol=1e-9)
    assert_values_close(rows["raw"], ref["raw"], sc["raw"], 1e-9, what="raw")
    A = ne.A[np.triu_indices(6)]
    np.testing.assert_allclose(A, ne_ref[:21], rtol=1e-9, atol=1e-9 * np.abs(ne_ref[:21]).max())
    np.testing.assert_allclose(ne.g, ne_ref[21:27], rtol=1e-9, atol=1e-9 * np.abs(ne_ref[21:27]).max())
    assert abs(ne.cost - ne_ref[27]) <= 1e-9 * abs(ne_ref[27])
    assert ne.valid == int(ne_ref[28])


# ---- K5-K8 update -----------------------------------------------------------------
def _split(obs, s, splits):
    m = len(obs.xy)
    chunk = m // splits
    b = s * chunk
    e = m if s == splits - 1 else b + chunk
    return T.TerrainObservation(obs.xy[b:e], obs.z[b:e])


@pytest.mark.parametrize("seed,n_points,mesh,cutoff,splits", [(26, 400, 0.15, 10.0, 8),
                                                               (27, 150, 0.2, 10.0, 1),
                                                               (23, 300, 0.12, 0.0, 4)])
def test_recursive_update_parity(gpu_ctx, seed, n_points, mesh, cutoff, splits):
    k, cs, obs = make_field(seed, n_points, mesh, cutoff)
    g, o = _models(k, cs)
    for s in range(splits):
        part = _split(obs, s, splits)
        rg = g.recursive_update(part, False)
        ro = o.recursive_update(part.xy, part.z, False)
        assert not rg.rejected and not ro["rejected"]
        assert (rg.active_blocks, rg.active_centers) == (ro["active_blocks"], ro["active_centers"])
    assert rel_norm(g.weights(), o.weights()) < 1e-8
    for b in range(o.num_blocks()):
        assert rel_norm(g.block_info_inverse(b), o.block_info_inverse(b)) < 1e-8


def test_recursive_update_information_form(gpu_ctx):
    # m > n selects the information-form solver
    xy, z = c1_inputs(20000)
    k = T.KernelParams()
    k.finalize()
    cs = T.select_centers(T.TerrainObservation(xy, z), ROI1, 0.07, 0.12, 3)
    g, o = _models(k, cs)
    rg = g.recursive_update(T.TerrainObservation(xy[:4000], z[:4000]), False)
    ro = o.recursive_update(xy[:4000], z[:4000], False)
    assert rg.solver == "information"
    assert rg.active_centers == ro["active_centers"]
    assert rel_norm(g.weights(), o.weights()) < 1e-8
    for b in range(o.num_blocks()):
        assert rel_norm(g.block_info_inverse(b), o.block_info_inverse(b)) < 1e-8


def test_birth_parity(gpu_ctx):
    kern = T.KernelParams(sigma=0.08, sigma_eps=0.05)
    kern.finalize()
    first = np.array([[0.3 + 0.01 * i, 0.5] for i in range(50)])
    roi = T.Rect((0.0, 0.0), (3.0, 1.0))
    cs = T.select_centers(T.TerrainObservation(first, np.full(50, 0.2)), roi, 0.1, 0.15, 3)
    g, o = _models(kern, cs)
    g.recursive_update(T.TerrainObservation(first, np.full(50, 0.2)))
    o.recursive_update(first, np.full(50, 0.2))
    second = np.array([[2.0 + 0.01 * i, 0.5] for i in range(50)])
    rg = g.recursive_update(T.TerrainObservation(second, np.full(50, 0.4)))
    ro = o.recursive_update(second, np.full(50, 0.4))
    assert rg.born_centers == ro["born_centers"] > 0
    assert np.array_equal(g.centers().centers, o.centers())
    assert np.array_equal(g.block_index(), o.block_index())
    assert rel_norm(g.weights(), o.weights()) < 1e-8
    q = g.predict_height([2.25, 0.5])
    assert q.supported and abs(q.z - 0.4) <= 0.04


def test_batch_fit_parity(gpu_ctx):
    k, cs, obs, g, o = _fitted_pair(seed=25, n_points=200, mesh=0.15, cutoff=10.0)
    assert rel_norm(g.weights(), o.weights()) < 1e-10
    for b in range(o.num_blocks()):
        assert rel_norm(g.block_info_inverse(b), o.block_info_inverse(b)) < 1e-9


def test_snapshot_byte_compatible(gpu_ctx, tmp_path):
    k, cs, obs, g, o = _fitted_pair(seed=28)
    pg, po = tmp_path / "g.bin", tmp_path / "o.bin"
    g.save(pg)
    # the oracle loads the device model's snapshot and vice versa
    o2 = orc.Model.load_file(pg)
    assert np.array_equal(o2.centers(), o.centers())
    o.save(po)
    g2 = T.TerrainModel.load(po)
    q = uniform_xy(orc.Rng(29), 20, 0.1, 0.9)
    z1, _, _, _ = g.predict(q)
    z2, _, _, _ = g2.predict(q)
    np.testing.assert_allclose(z1, z2, rtol=1e-10)
    g.save(pg)
    g3 = T.TerrainModel.load(pg)
    z3, _, _, _ = g3.predict(q)
    assert np.array_equal(z3, z1)


# ---- lattice fast path edge cases + scans -------------------------------------
def _lattice_model_with_holes(seed=41):
    """C1-like lattice model with holes (absent nodes) and ragged support."""
    xy, z = c1_inputs(6000, seed)
    keep = ~((xy[:, 0] > 0.3) & (xy[:, 0] < 0.5) & (xy[:, 1] > 0.4) & (xy[:, 1] < 0.7))
    xy, z = xy[keep], z[keep]
    k = T.KernelParams()
    k.finalize()
    cs = T.select_centers(T.TerrainObservation(xy, z), ROI1, 0.07, 0.12, 3)
    g, o = _models(k, cs)
    w = np.cos(np.arange(len(cs.centers)) * 0.71)
    g.set_weights(w)
    o.set_weights(w)
    return k, cs, g, o


def test_lattice_edges_and_holes(gpu_ctx):
    k, cs, g, o = _lattice_model_with_holes()
    rng = orc.Rng(43)
    q = uniform_xy(rng, 20000, -0.5, 1.6)
    # points exactly on nodes and on the cutoff circle around nodes
    c = cs.centers[::7]
    ang = np.linspace(0, 2 * np.pi, len(c), endpoint=False)
    ring = c + k.cutoff_radius * np.stack([np.cos(ang), np.sin(ang)], 1)
    axis = c + np.stack([np.full(len(c), k.cutoff_radius), np.zeros(len(c))], 1)
    q = np.concatenate([q, c, ring, axis])
    z, s, gx, gy = g.predict(q)
    zr, sr, gxr, gyr = o.predict(q)
    assert np.array_equal(s, sr)
    hs, gs = scales(o, q, k.sigma)
    assert_values_close(z, zr, hs, what="height")
    assert_values_close(gx, gxr, gs, what="gx")
    assert_values_close(gy, gyr, gs, what="gy")


def test_scan_rows_equal_unbinned(gpu_ctx):
    k, cs, g, o = _lattice_model_with_holes(45)
    R = so3_exp([0.03, -0.02, 0.5])
    t = np.array([0.2, 0.1, 0.3])
    pts = np.concatenate([uniform_xy(orc.Rng(46), 30000, -0.2, 1.3), np.full((30000, 1), 0.02)], 1)
    h = (pts - t) @ R
    rows, ne = kin.manifold_rows(g, R, t, h, 0.0, 1.0, 0.05, want=("r", "J", "valid"))
    sc = kin.Scan(g, so3_exp([0.0, 0.0, 0.45]), t + 0.05, h)
    perm = sc.permutation()
    assert np.array_equal(np.sort(perm), np.arange(len(h)))
    srows, sne = sc.manifold_rows(R, t, 0.0, 1.0, 0.05)
    assert np.array_equal(srows["valid"], rows["valid"][perm])
    assert np.array_equal(srows["r"], rows["r"][perm])  # same per-point arithmetic
    Jn = rows["J"].reshape(6, -1)
    Js = srows["J"].reshape(6, -1)
    assert np.array_equal(Js, Jn[:, perm])
    np.testing.assert_allclose(sne.A, ne.A, rtol=1e-12, atol=1e-12 * np.abs(ne.A).max())
    assert sne.valid == ne.valid


def test_generic_path_random_centres(gpu_ctx):
    # non-lattice centres (acceptance_main.cpp:121-127 style) use the generic sweep
    rng = orc.Rng(102)
    c = uniform_xy(rng, 300, 0.0, 2.0)
    k = T.KernelParams(sigma=0.08, sigma_eps=0.05)
    k.finalize()
    cs = T.CenterSet(c, 0.07, 0.12, 3, T.Rect((0.0, 0.0), (2.0, 2.0)))
    g, o = _models(k, cs)
    w = np.sin(np.arange(300) * 1.3)
    g.set_weights(w)
    o.set_weights(w)
    q = uniform_xy(orc.Rng(103), 5000, -0.3, 2.3)
    z, s, gx, gy = g.predict(q)
    zr, sr, gxr, gyr = o.predict(q)
    assert np.array_equal(s, sr)
    hs, gs = scales(o, q, k.sigma)
    assert_values_close(z, zr, hs, what="height")
    assert_values_close(gx, gxr, gs, what="gx")


def test_generic_fine_grid_binned_manifold_rows(gpu_ctx):
    """Non-lattice centres (a jittered mesh) on a scan-binned evaluation:
    the fine-grid generic sweep (warp-union candidate cells) against the
    oracle's rows, bit-exact validity and the §8d scales."""
    rng = np.random.default_rng(61)
    side = 1.6
    nodes = np.arange(int(side / 0.07) + 1) * 0.07
    gx, gy = np.meshgrid(nodes, nodes, indexing="ij")
    c = np.stack([gx.ravel(), gy.ravel()], 1) + rng.uniform(-0.004, 0.004, (gx.size, 2))
    k = T.KernelParams()
    k.finalize()
    cs = T.CenterSet(c, 0.07, 0.12, 3, T.Rect((0.0, 0.0), (side, side)))
    g, o = _models(k, cs)
    assert g.sweep()[0] == 0  # generic
    w = 0.05 * np.sin(3.0 * c[:, 0]) * np.cos(2.0 * c[:, 1])
    g.set_weights(w)
    o.set_weights(w)
    R = so3_exp([0.01, -0.02, 0.3])
    t = np.array([0.05, -0.03, 0.02])
    pts = np.c_[rng.uniform(-0.1, side + 0.1, (40_000, 2)), rng.normal(0, 0.03, 40_000)]
    h = (pts - t) @ R
    scan = kin.Scan(g, R, t, h)
    srows, sne = scan.manifold_rows(R, t, 0.0, 1.0, 0.05)
    rows, ne = kin.manifold_rows(g, R, t, h, 0.0, 1.0, 0.05)
    ref, ne_ref = o.manifold_rows(R, t, h, 0.0, 1.0, 0.05)
    assert np.array_equal(rows["valid"], ref["valid"])
    sc = manifold_row_scales(o, R, t, h, ref["J"])
    assert_manifold_rows_close(rows["r"], rows["J"].reshape(6, -1).T, ref["r"], ref["J"], sc, rtol=1e-9)
    perm = scan.permutation()
    assert np.array_equal(srows["valid"], ref["valid"][perm])
    np.testing.assert_allclose(sne.A, ne.A, rtol=1e-10, atol=1e-10 * np.abs(ne.A).max())
