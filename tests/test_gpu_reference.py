"""GPU vs THE REFERENCE ITSELF (oracle/_ref: the unchanged reference sources
compiled here) on the benchmarked update configurations and failure paths.

* C3 (64 x 64 = 4,096 centres, staircase), m = 400: the one-shot Woodbury
  formulation on the device vs the reference's chunk-64 Woodbury.
* n > 1024 with m > n: the information form (64-wide lookahead Cholesky,
  banded X = L^-1) vs the same reference algorithm.
* C4 at reduced M (a 96 x 96 bumps lattice, 1 m footprint).
* a 30-scan stream with births: reports exact, weights / info_inv per scan.
* rejected = true (non-PD innovation, terrain_model.cpp:222-230): births
  persist, weights and blocks untouched.

Bars: reports, centres and block ids exact; weights and
info_inv within 1e-8 relative (norm), the reference's acceptance bar.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle as orc
from helpers import rel_norm
from paper_2509_26222_b200 import terrain as T

REF = orc.reference()
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(REF is None, reason="oracle/_ref not built")]

RES, RA, CNT = 0.07, 0.12, 3


def staircase(x):
    """TerrainSpec::staircase(0.08, 0.5, 10, x0 = 0.5) (terrain_spec.cpp:72-77)."""
    xr = x - 0.5
    return np.where(xr < 0.0, 0.0, 0.08 * np.minimum(np.floor(xr / 0.5), 10.0))


def bumps(x, y):
    return 0.05 * np.sin(2 * np.pi * x / 1.5) * np.sin(2 * np.pi * y / 1.5)


def kernel():
    k = T.KernelParams()
    k.finalize()
    return k


def lattice(side, seed):
    roi = T.Rect((0.0, 0.0), (side, side))
    rng = np.random.default_rng(seed)
    sup = rng.uniform(0.0, side, (int(side * side * 1500), 2))
    nodes = REF.supported_mesh_nodes(sup, np.zeros(len(sup)), roi, RES, RA, CNT)
    return T.CenterSet(nodes, RES, RA, CNT, roi)


def compare_models(g, r, what, tol=1e-8):
    assert g.num_centers() == r.num_centers(), what
    assert np.array_equal(g.centers().centers.view(np.uint64), r.centers().view(np.uint64)), what
    assert np.array_equal(g.block_index(), r.block_index()), what
    e_w = rel_norm(g.weights(), r.weights())
    e_i = max(rel_norm(g.block_info_inverse(b), r.block_info_inverse(b)) for b in range(r.num_blocks()))
    print(f"[parity] {what}: weights {e_w:.2e}, info_inv {e_i:.2e} (bar {tol:g})")
    assert e_w <= tol, f"{what}: weights rel err {e_w:.3e}"
    assert e_i <= tol, f"{what}: info_inv rel err {e_i:.3e}"
    return e_w, e_i


def update_both(g, r, xy, z, birth=True):
    rg = g.recursive_update(T.TerrainObservation(xy, z), birth)
    rr = r.recursive_update(xy, z, birth)
    assert (rg.active_blocks, rg.active_centers, rg.born_centers, rg.rejected) == (
        rr["active_blocks"], rr["active_centers"], rr["born_centers"], rr["rejected"])
    return rg


def test_c3_woodbury_n4096_m400(gpu_ctx):
    cs = lattice(4.41, 3)
    assert len(cs.centers) == 4096
    k = kernel()
    g, r = T.TerrainModel(k, cs), REF.Model(k, cs)
    rng = np.random.default_rng(7)
    clean = rng.uniform(0.0, 4.41, (400, 2))
    xy = clean + rng.normal(0.0, 0.1, clean.shape)
    rep = update_both(g, r, xy, staircase(clean[:, 0]), False)
    assert rep.active_centers == 4096 and rep.solver.startswith("woodbury"), rep
    compare_models(g, r, "C3 m=400")


def test_information_form_n_gt_1024(gpu_ctx):
    cs = lattice(2.52, 5)            # 37 x 37 = 1,369 centres
    k = kernel()
    g, r = T.TerrainModel(k, cs), REF.Model(k, cs)
    rng = np.random.default_rng(8)
    clean = rng.uniform(0.0, 2.52, (1600, 2))
    xy = clean + rng.normal(0.0, 0.1, clean.shape)
    rep = update_both(g, r, xy, staircase(clean[:, 0] + 1.0), False)
    assert rep.active_centers > 1024 and 1600 > rep.active_centers and rep.solver.startswith("info"), rep
    compare_models(g, r, "info form n>1024")
    # a second scan on top (the updated blocks become the prior)
    clean = rng.uniform(0.0, 2.52, (1500, 2))
    xy = clean + rng.normal(0.0, 0.1, clean.shape)
    update_both(g, r, xy, staircase(clean[:, 0] + 1.0), False)
    compare_models(g, r, "info form, second scan")


def test_c4_reduced_footprint(gpu_ctx):
    cs = lattice(6.72, 6)             # 97 x 97 bumps lattice
    k = kernel()
    g, r = T.TerrainModel(k, cs), REF.Model(k, cs)
    rng = np.random.default_rng(9)
    for step in range(2):
        cx, cy = 3.0 + 0.4 * step, 3.2 + 0.3 * step
        rad = 1.0 * np.sqrt(rng.uniform(0, 1, 1200))
        a = rng.uniform(0, 2 * np.pi, 1200)
        clean = np.stack([cx + rad * np.cos(a), cy + rad * np.sin(a)], 1)
        xy = clean + rng.normal(0.0, 0.02, clean.shape)
        update_both(g, r, xy, bumps(clean[:, 0], clean[:, 1]), False)
        compare_models(g, r, f"C4 reduced, scan {step}")


def test_stream_30_scans_with_births(gpu_ctx):
    """C2-like: the model starts empty and grows through births along a path;
    every scan's report, centres, block ids, weights and info_inv."""
    roi = T.Rect((0.0, 0.0), (6.0, 3.0))
    k = kernel()
    empty = T.CenterSet(np.zeros((0, 2)), RES, RA, CNT, roi)
    g, r = T.TerrainModel(k, empty), REF.Model(k, empty)
    rng = np.random.default_rng(11)
    worst = (0.0, 0.0)
    for s in range(30):
        x0 = 0.3 + 0.15 * s
        clean = np.stack([rng.uniform(x0 - 0.5, x0 + 0.5, 200), rng.uniform(0.8, 2.2, 200)], 1)
        xy = clean + rng.normal(0.0, 0.01, clean.shape)
        update_both(g, r, xy, staircase(clean[:, 0]), True)
        e = compare_models(g, r, f"stream scan {s}")
        worst = tuple(max(a, b) for a, b in zip(worst, e))
    assert g.num_centers() > 300
    print(f"30-scan stream: worst weights {worst[0]:.2e}, info_inv {worst[1]:.2e}")


def test_rejected_update_keeps_model_but_births_persist(gpu_ctx, tmp_path):
    """terrain_model.cpp:222-230: a non-PD innovation rejects the update
    after births were applied; weights and existing blocks are untouched."""
    side = 1.4
    full = lattice(side, 12)
    keep = full.centers[:, 0] <= 0.8 + 1e-9          # the x > 0.8 nodes get born later
    cs = T.CenterSet(full.centers[keep], RES, RA, CNT, full.roi)
    k = kernel()
    g, r = T.TerrainModel(k, cs), REF.Model(k, cs)
    rng = np.random.default_rng(13)
    clean = rng.uniform(0.1, 0.7, (300, 2))
    update_both(g, r, clean, staircase(clean[:, 0] + 0.6), False)
    # poison block 0's info_inv: strongly negative definite
    bn = len(r.block_members(0))
    bad = -1e3 * np.eye(bn)
    g.set_block_info_inverse(0, bad)
    r.set_block_info_inverse(0, bad)
    w_before = g.weights().copy()
    blocks_before = [g.block_info_inverse(b).copy() for b in range(g.num_blocks())]
    # a few points over block 0 plus a strip beyond the centres (births);
    # m stays below the active count so both sides run the Woodbury innovation
    c0 = r.centers()[r.block_members(0)].mean(0)
    pts = np.concatenate([c0 + rng.uniform(-0.15, 0.15, (25, 2)),
                          np.stack([rng.uniform(1.0, 1.2, 25), rng.uniform(0.3, 0.6, 25)], 1)])
    rep = update_both(g, r, pts, np.zeros(len(pts)), True)
    assert rep.rejected and rep.born_centers > 0, rep
    assert np.array_equal(g.centers().centers.view(np.uint64), r.centers().view(np.uint64))
    n0 = len(w_before)
    assert np.array_equal(g.weights()[:n0], w_before) and np.all(g.weights()[n0:] == 0.0)
    assert rel_norm(g.weights(), r.weights()) <= 1e-8
    for b, a in enumerate(blocks_before):
        gb = g.block_info_inverse(b)
        if gb.shape == a.shape:
            assert np.array_equal(gb, a), b


def test_kernel_eval_matches_reference(gpu_ctx):
    """tlg_kernel_eval vs the reference's kernel_eval (kernel.cpp:27-35):
    the exact zero beyond the cutoff bit for bit, values to 1e-15 relative
    (device exp vs glibc exp), domain errors alike."""
    k = T.KernelParams()
    k.finalize()
    rng = np.random.default_rng(21)
    x = rng.uniform(-0.5, 0.5, (4000, 2))
    c = rng.uniform(-0.5, 0.5, (4000, 2))
    # pairs straddling the cutoff within an ulp
    d = np.array([k.cutoff_radius, np.nextafter(k.cutoff_radius, 0), np.nextafter(k.cutoff_radius, 1)])
    x = np.concatenate([x, np.stack([d, np.zeros(3)], 1)])
    c = np.concatenate([c, np.zeros((3, 2))])
    for bw in (k.sigma, k.sigma_tilde(), 0.3):
        got = T.kernel_eval(k, x, c, bw)
        ref = np.array([REF.kernel_eval(k, xi, ci, bw) for xi, ci in zip(x, c)])
        assert np.array_equal(got == 0.0, ref == 0.0)
        np.testing.assert_allclose(got, ref, rtol=1e-15, atol=0)
    with pytest.raises(T.DomainError):
        T.kernel_eval(k, np.array([[np.nan, 0.0]]), np.zeros((1, 2)), 0.04)
    with pytest.raises(T.DomainError):
        T.kernel_eval(k, np.zeros((1, 2)), np.zeros((1, 2)), -1.0)
