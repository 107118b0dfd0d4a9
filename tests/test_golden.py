"""Golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py
from the reference itself, oracle/_ref). CPU: the plain-C++ restatement
reproduces them (bit-exact for indexing, within the reference's own 1e-10 bar
for Eigen arithmetic). GPU: the sm_100a path matches them with no oracle at
run time, at the SURVEY §8d tolerances."""
from pathlib import Path

import numpy as np
import pytest

import oracle as orc
from helpers import assert_manifold_rows_close, assert_values_close
from paper_2509_26222_b200.terrain import CenterSet, KernelParams, Rect

G = Path(__file__).resolve().parent / "golden"
ROI1 = Rect((0.0, 0.0), (1.05, 1.05))


def load(name):
    return dict(np.load(G / name))


def _kernel(a):
    return KernelParams(*map(float, a["kernel"]))


# ---- CPU: oracle reproduces the fixtures --------------------------------------
def test_oracle_select_golden():
    d = load("select_c1.npz")
    nodes = orc.supported_mesh_nodes(d["xy"], d["z"], ROI1, 0.07, 0.12, 3, True)
    assert np.array_equal(nodes.view(np.uint64), d["nodes"].view(np.uint64))


def test_oracle_eval_golden():
    d = load("eval_field.npz")
    cs = CenterSet(d["centers"], *d["mesh"][:2], int(d["mesh"][2]), Rect((0.0, 0.0), (1.0, 1.0)))
    m = orc.fit_batch_ridge(_kernel(d), cs, d["obs_xy"], d["obs_z"])
    assert np.linalg.norm(m.weights() - d["weights"]) <= 1e-10 * np.linalg.norm(d["weights"])
    m.set_weights(d["weights"])  # then evaluation is bit-for-bit the reference's
    z, s, gx, gy = m.predict(d["q"])
    assert np.array_equal(s, d["sup"])
    assert np.array_equal(z, d["z"]) and np.array_equal(gx, d["gx"]) and np.array_equal(gy, d["gy"])


def test_oracle_update_golden():
    d = load("update.npz")
    cs = CenterSet(d["centers"], 0.15, 0.15, 3, Rect((0.0, 0.0), (1.0, 1.0)))
    m = orc.Model(_kernel(d), cs)
    for s in range(4):
        r = m.recursive_update(d["obs_xy"][s * 100:(s + 1) * 100], d["obs_z"][s * 100:(s + 1) * 100],
                               False)
        assert [r["active_blocks"], r["active_centers"], r["born_centers"], r["rejected"]] == \
            list(d["reports"][s])
    assert np.linalg.norm(m.weights() - d["weights"]) <= 1e-10 * np.linalg.norm(d["weights"])


# ---- GPU: device path vs fixtures ------------------------------------------------
@pytest.mark.gpu
def test_gpu_matches_golden(gpu_ctx):
    from paper_2509_26222_b200 import kinematics as kin
    from paper_2509_26222_b200 import terrain as T

    d = load("select_c1.npz")
    cs = T.select_centers(T.TerrainObservation(d["xy"], d["z"]), ROI1, 0.07, 0.12, 3)
    assert np.array_equal(cs.centers.view(np.uint64), d["nodes"].view(np.uint64))

    e = load("eval_field.npz")
    cs = CenterSet(e["centers"], *e["mesh"][:2], int(e["mesh"][2]), Rect((0.0, 0.0), (1.0, 1.0)))
    g = T.fit_batch_ridge(_kernel(e), cs, T.TerrainObservation(e["obs_xy"], e["obs_z"]))
    w = g.weights()
    assert np.linalg.norm(w - e["weights"]) <= 1e-8 * np.linalg.norm(e["weights"])
    g.set_weights(e["weights"])  # evaluate the golden weights exactly
    z, s, gx, gy = g.predict(e["q"])
    assert np.array_equal(s, e["sup"])
    assert_values_close(z, e["z"], e["scale_z"], 1e-9, what="z")
    assert_values_close(gx, e["gx"], e["scale_g"], 1e-9, what="gx")
    assert_values_close(gy, e["gy"], e["scale_g"], 1e-9, what="gy")

    mf = load("manifold.npz")
    rows, ne = kin.manifold_rows(g, mf["R"], mf["t"], mf["h"], 0.0, 1.0, 0.05,
                                 want=("r", "J", "valid"))
    assert np.array_equal(rows["valid"], mf["valid"])
    # 1e-9 of max(|ref|, the row's sum |w kappa| scale), no floor
    sc = {"r": mf["scale_r"], "J": list(mf["scale_J"].T)}
    assert_manifold_rows_close(rows["r"], rows["J"].reshape(6, -1).T, mf["r"],
                               mf["J"].reshape(-1, 6), sc, rtol=1e-9)
    np.testing.assert_allclose(ne.A[np.triu_indices(6)], mf["ne"][:21], rtol=1e-9, atol=1e-9)

    u = load("update.npz")
    cs = CenterSet(u["centers"], 0.15, 0.15, 3, Rect((0.0, 0.0), (1.0, 1.0)))
    gu = T.TerrainModel(_kernel(u), cs)
    for s_ in range(4):
        r = gu.recursive_update(T.TerrainObservation(u["obs_xy"][s_ * 100:(s_ + 1) * 100],
                                                     u["obs_z"][s_ * 100:(s_ + 1) * 100]), False)
        assert [r.active_blocks, r.active_centers, r.born_centers, int(r.rejected)] == \
            list(u["reports"][s_])
    assert np.linalg.norm(gu.weights() - u["weights"]) <= 1e-8 * np.linalg.norm(u["weights"])
    for b in range(gu.num_blocks()):
        ref = u[f"info_inv_{b}"]
        assert np.linalg.norm(gu.block_info_inverse(b) - ref) <= 1e-8 * np.linalg.norm(ref)
