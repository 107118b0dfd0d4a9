"""Batch-predict consumers: select_ground_points
(pipeline.cpp:150-170), terrain_error_histogram (metrics.cpp:199-232) and
export_csv (terrain_model.cpp:255-267) on the device vs the CPU oracle —
kept points, their order and histogram counts bit-exact."""
import numpy as np
import pytest

import oracle as orc
from helpers import make_field, so3_exp
from paper_2509_26222_b200 import consumers as K
from paper_2509_26222_b200 import terrain as T


def _scan(seed, n):
    rng = np.random.default_rng(seed)
    p = rng.uniform(-3.0, 3.0, size=(n, 3))
    p[:, 2] *= 0.2
    kinds = rng.integers(0, 3, n).astype(np.uint8)
    # exact voxel / ROI / radius boundaries
    p[:50, 0] = np.round(p[:50, 0] / 0.12) * 0.12
    p[50:80, 1] = 0.0
    return p, kinds


def test_oracle_ground_points_rules():
    # hand-checked case: duplicate voxel, non-ground, outside ROI, outside radius
    p = np.array([[0.05, 0.05, 0.1], [0.06, 0.07, 0.2], [0.5, 0.5, 0.3], [5.0, 0.1, 0.0],
                  [0.3, 0.3, 0.4], [1.9, 1.9, 0.0]])
    kinds = np.array([2, 2, 0, 2, 2, 2], dtype=np.uint8)
    xy, z = orc.select_ground_points(p, kinds, np.eye(3), [0.0, 0.0, 0.0],
                                     T.Rect((0.0, 0.0), (2.0, 2.0)), 2.5, 0.12, 400)
    assert np.array_equal(z, [0.1, 0.4])  # 2nd: same voxel; 3rd: edge; 4th: ROI; 6th: radius
    xy, z = orc.select_ground_points(p, kinds, np.eye(3), [0.0, 0.0, 0.0],
                                     T.Rect((0.0, 0.0), (2.0, 2.0)), 2.5, 0.12, 1)
    assert np.array_equal(z, [0.1])


@pytest.mark.gpu
@pytest.mark.parametrize("seed,n,cap", [(1, 5000, 400), (2, 200000, 20000), (3, 300, 5)])
def test_select_ground_points_parity(gpu_ctx, seed, n, cap):
    p, kinds = _scan(seed, n)
    R = so3_exp([0.01, 0.02, 0.7])
    t = np.array([0.3, -0.2, 0.5])
    roi = T.Rect((-1.0, -1.5), (2.0, 2.2))
    obs = K.select_ground_points(p, kinds, R, t, roi, 2.5, 0.12, cap)
    xy, z = orc.select_ground_points(p, kinds, R, t, roi, 2.5, 0.12, cap)
    assert np.array_equal(np.asarray(obs.xy).view(np.uint64), xy.view(np.uint64))
    assert np.array_equal(np.asarray(obs.z).view(np.uint64), z.view(np.uint64))


@pytest.mark.gpu
@pytest.mark.parametrize("trim,bins", [(0.0, 25), (0.1, 25), (0.37, 7)])
def test_error_histogram_parity(gpu_ctx, trim, bins):
    k, cs, obs = make_field(51, 400)
    g = T.fit_batch_ridge(k, cs, obs)
    o = orc.fit_batch_ridge(k, cs, obs.xy, obs.z)
    rng = np.random.default_rng(7)
    xy = rng.uniform(-0.2, 1.2, size=(30000, 2))
    z = 0.1 * np.sin(4.0 * xy[:, 0]) + 0.05 * xy[:, 1] ** 2 + rng.normal(0, 0.05, 30000)
    h = K.terrain_error_histogram(g, xy, z, trim, bins)
    r = o.error_histogram(xy, z, trim, bins)
    assert np.array_equal(h.edges, r["edges"])
    assert h.trimmed == r["trimmed"] and h.overflow == r["overflow"]
    # counts: bin edges are exact; errors agree to ~1e-15, so only samples
    # within rounding of an edge could move (none expected at these sizes)
    assert np.array_equal(h.counts, r["counts"].astype(np.uint64))
    assert h.total() == 30000 - h.trimmed


@pytest.mark.gpu
def test_error_histogram_errors(gpu_ctx):
    k, cs, obs = make_field(52, 200)
    g = T.TerrainModel(k, cs)
    with pytest.raises(T.InvalidArgument):
        K.terrain_error_histogram(g, np.zeros((0, 2)), np.zeros(0))
    with pytest.raises(T.InvalidArgument):
        K.terrain_error_histogram(g, np.zeros((3, 2)), np.zeros(3), 1.0)


@pytest.mark.gpu
def test_export_csv_matches_oracle(gpu_ctx, tmp_path):
    k, cs, obs = make_field(53, 400)
    g = T.fit_batch_ridge(k, cs, obs)
    o = orc.fit_batch_ridge(k, cs, obs.xy, obs.z)
    gx, gy, gz = K.export_grid(g, 0.013)
    rx, ry, rz = o.export_grid(0.013)
    assert np.array_equal(gx, rx) and np.array_equal(gy, ry)
    np.testing.assert_allclose(gz, rz, rtol=1e-9, atol=1e-12)
    path = tmp_path / "grid.csv"
    g.export_csv(str(path), 0.013)
    lines = path.read_text().splitlines()
    assert lines[0] == "x,y,z_pred" and len(lines) == len(rx) + 1
