"""Is the C5 band Cholesky work- or chain-bound? Same 316 x 316 lattice
(3,121 32-row tile steps) with a narrower kernel: the band (and the work,
~bwt^2) shrinks while the tile chain stays. Prints the stage trace."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2509_26222_b200 import terrain as T  # noqa: E402

for sigma in (0.04, 0.025, 0.015):
    side = 315 * 0.07
    nodes = np.arange(316) * 0.07
    gx, gy = np.meshgrid(nodes, nodes, indexing="ij")
    cs = T.CenterSet(np.stack([gx.ravel(), gy.ravel()], 1), 0.07, 0.12, 3,
                     T.Rect((0.0, 0.0), (side, side)))
    k = T.KernelParams(sigma=sigma, sigma_eps=sigma * 2.5)
    k.finalize()
    rng = np.random.default_rng(1)
    xy = rng.uniform(0, side, (2_000_000, 2))
    z = 0.05 * np.sin(xy[:, 0])
    m = T.TerrainModel(k, cs)
    n, ld, el = m.batch_system()
    print(f"sigma {sigma}: cutoff {k.cutoff_radius:.3f} ld {ld}", flush=True)
    for _ in range(2):
        T.fit_batch_ridge(k, cs, T.TerrainObservation(xy, z))
    torch.cuda.synchronize()
