"""Generates the golden fixtures in this directory from THE REFERENCE ITSELF
(oracle/_ref: the unchanged /root/reference sources compiled by `make -C
oracle ref`, driven through oracle.reference()), falling back to the CPU
restatement only where the reference is not built. Each fixture records its
`source`; tests/test_reference_pin.py pins the restatement to the reference.
Run here (needs /root/reference): python tests/golden/make_golden.py

Fixtures (npz):
  select_c1.npz   C1 inputs (20k noisy points, seed 2509) -> node list (bits)
  eval_field.npz  fitted make_field(23) model + 600 queries -> z, supported, grad
  manifold.npz    same model, bench pose, 600 lever arms -> rows + normal eqs
  update.npz      make_field(26, 400, 0.15, cutoff 10) over 4 recursive splits
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path[:0] = [str(HERE.parent), str(HERE.parent.parent), str(HERE.parent.parent / "oracle")]

import oracle as orc  # noqa: E402
from helpers import c1_inputs, make_field, manifold_row_scales, uniform_xy  # noqa: E402
from paper_2509_26222_b200.terrain import Rect  # noqa: E402

ROI1 = Rect((0.0, 0.0), (1.05, 1.05))


def model_arrays(m):
    nb = m.num_blocks()
    return dict(weights=m.weights(), block_index=m.block_index(),
                **{f"info_inv_{b}": m.block_info_inverse(b) for b in range(nb)})


def main():
    ref = orc.reference() or orc
    src = ref.BACKEND
    xy, z = c1_inputs(20000)
    nodes = ref.supported_mesh_nodes(xy, z, ROI1, 0.07, 0.12, 3, True)
    np.savez_compressed(HERE / "select_c1.npz", xy=xy, z=z, nodes=nodes, source=src)

    k, cs, obs = make_field(23)
    m = ref.fit_batch_ridge(k, cs, obs.xy, obs.z)
    q = uniform_xy(orc.Rng(24), 600, -0.2, 1.2)
    zq, s, gx, gy = m.predict(q)
    np.savez_compressed(HERE / "eval_field.npz", kernel=[k.sigma, k.sigma_eps, k.lambda_,
                                                        k.cutoff_radius],
                        centers=np.asarray(cs.centers), mesh=[cs.mesh_resolution,
                                                               cs.accept_radius, cs.accept_count],
                        obs_xy=obs.xy, obs_z=obs.z, q=q, z=zq, sup=s, gx=gx, gy=gy,
                        scale_z=m.scales(q)[0], scale_g=m.scales(q)[1], source=src,
                        **model_arrays(m))

    R = ref.so3_exp([0.02, -0.015, 0.04])
    t = np.array([0.1, -0.05, 0.08])
    pts = np.concatenate([uniform_xy(orc.Rng(7), 600, -0.1, 1.1), np.full((600, 1), 0.05)], 1)
    h = (pts - t) @ R
    rows, ne = m.manifold_rows(R, t, h, 0.0, 1.0, 0.05)
    sc = manifold_row_scales(m, R, t, h, rows["J"])
    np.savez_compressed(HERE / "manifold.npz", R=R, t=t, h=h, r=rows["r"], J=rows["J"],
                        valid=rows["valid"], raw=rows["raw"], ne=ne, scale_r=sc["r"],
                        scale_raw=sc["raw"], scale_J=np.stack(sc["J"], 1), source=src)

    k2, cs2, obs2 = make_field(26, 400, 0.15, 10.0)
    mu = ref.Model(k2, cs2)
    reps = []
    for s_ in range(4):
        b, e = s_ * 100, (s_ + 1) * 100
        r = mu.recursive_update(obs2.xy[b:e], obs2.z[b:e], False)
        reps.append([r["active_blocks"], r["active_centers"], r["born_centers"], r["rejected"]])
    np.savez_compressed(HERE / "update.npz", kernel=[k2.sigma, k2.sigma_eps, k2.lambda_,
                                                    k2.cutoff_radius],
                        centers=np.asarray(cs2.centers), obs_xy=obs2.xy, obs_z=obs2.z,
                        reports=np.array(reps), source=src, **model_arrays(mu))
    print(f"golden fixtures ({src}) written to", HERE)


if __name__ == "__main__":
    main()
