"""Shared synthetic-input generators (std::mt19937_64 via the oracle's RNG so
inputs follow the reference tests' seeds and distributions) and tolerance
checks used by the parity tests."""
from __future__ import annotations

import math

import numpy as np

import oracle as orc
from paper_2509_26222_b200.terrain import CenterSet, KernelParams, Rect, TerrainObservation


def uniform_xy(rng: orc.Rng, n, lo, hi, lo_y=None, hi_y=None):
    lo_y = lo if lo_y is None else lo_y
    hi_y = hi if hi_y is None else hi_y
    out = np.empty((n, 2))
    for i in range(n):
        out[i, 0] = rng.uniform(lo, hi)
        out[i, 1] = rng.uniform(lo_y, hi_y)
    return out


def make_field(seed, n_points=300, mesh=0.12, cutoff=0.0):
    """test_terrain_model.cpp:21-38 (random smooth surface on [0,1]^2)."""
    rng = orc.Rng(seed)
    k = KernelParams(sigma=0.08, sigma_eps=0.05, cutoff_radius=cutoff)
    k.cutoff_radius = orc.kernel_finalize(k)
    xy = uniform_xy(rng, n_points, 0.0, 1.0)
    z = 0.1 * np.sin(4.0 * xy[:, 0]) + 0.05 * xy[:, 1] * xy[:, 1]
    roi = Rect((0.0, 0.0), (1.0, 1.0))
    nodes = orc.supported_mesh_nodes(xy, z, roi, mesh, 0.15, 3, throw_empty=True)
    cs = CenterSet(nodes, mesh, 0.15, 3, roi)
    return k, cs, TerrainObservation(xy, z)


def c1_inputs(n_points=20000, seed=2509):
    """16x16 lattice on [0,1.05]^2, 20k noisy points."""
    rng = orc.Rng(seed)
    nd = orc.Normal(0.0, 0.1)
    clean = np.empty((n_points, 2))
    noisy = np.empty((n_points, 2))
    for i in range(n_points):
        clean[i, 0] = rng.uniform(0.0, 1.05)
        clean[i, 1] = rng.uniform(0.0, 1.05)
        noisy[i, 0] = clean[i, 0] + nd.draw(rng)
        noisy[i, 1] = clean[i, 1] + nd.draw(rng)
    z = 0.1 * np.sin(4.0 * clean[:, 0]) + 0.05 * clean[:, 1] ** 2
    return noisy, z


def so3_exp(w):
    return orc.so3_exp(w)


def assert_values_close(got, ref, scale, rtol=1e-9, what="value"):
    """|got - ref| <= rtol * max(|ref|, scale) elementwise."""
    got, ref, scale = map(lambda a: np.asarray(a, dtype=np.float64), (got, ref, scale))
    bound = rtol * np.maximum(np.abs(ref), scale)
    err = np.abs(got - ref)
    bad = err > bound
    if bad.any():
        i = int(np.argmax(err - bound))
        raise AssertionError(f"{what}: {bad.sum()} entries out of tolerance; worst idx {i}: "
                             f"got {got.flat[i]!r} ref {ref.flat[i]!r} bound {bound.flat[i]:.3e}")


def rel_norm(a, b):
    a, b = np.asarray(a), np.asarray(b)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def scales(model_oracle, xy, sigma):
    w = model_oracle.weights()
    c = model_oracle.centers()
    hs = np.zeros(len(xy))
    gs = np.zeros(len(xy))
    for i, q in enumerate(xy):
        ids = model_oracle.centers_near(q)
        if len(ids) == 0:
            continue
        d = c[ids] - q
        d2 = (d ** 2).sum(1)
        k = np.exp(-d2 / (2 * sigma * sigma))
        hs[i] = np.abs(w[ids] * k).sum()
        gs[i] = (np.abs(w[ids] * k) * np.sqrt(d2)).sum() / (sigma * sigma)
    return hs, gs


def manifold_row_scales(model_oracle, R, t, h, ref_J):
    """Per-row parity scales of the manifold rows (1e-9 of
    max(|ref|, scale), scale built from sum |w kappa| of the same point):
    r ~ s S0 and J3, J4 ~ s S1 with S0 = sum |w kappa|, S1 = sum |w kappa| d /
    sigma^2, J0..J2 = s h x (R^T [-g, 1]) ~ s |h| S1, J5 = s exactly; s =
    sqrt(lambda_M) w_Huber = ref J5. No additive floor."""
    h = np.asarray(h, dtype=np.float64).reshape(-1, 3)
    xy = (h @ np.asarray(R).T + np.asarray(t))[:, :2]
    S0, S1 = model_oracle.scales(xy)
    s = np.abs(np.asarray(ref_J)[:, 5])
    hn = np.linalg.norm(h, axis=1)
    tiny = np.finfo(np.float64).tiny
    return {"r": s * S0 + tiny, "raw": S0 + tiny,
            "J": [s * hn * S1 + tiny] * 3 + [s * S1 + tiny] * 2 + [s + tiny]}


def assert_manifold_rows_close(got_r, got_J, ref_r, ref_J, sc, rtol=1e-9):
    """got_J, ref_J: (n, 6) row-major."""
    assert_values_close(got_r, ref_r, sc["r"], rtol, what="r")
    for c in range(6):
        assert_values_close(got_J[:, c], ref_J[:, c], sc["J"][c], rtol, what=f"J{c}")


__all__ = ["uniform_xy", "make_field", "c1_inputs", "so3_exp", "assert_values_close",
           "rel_norm", "scales", "math", "manifold_row_scales", "assert_manifold_rows_close"]
