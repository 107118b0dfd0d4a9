"""C4: M = 65,536 centres (256 x 256 lattice on [0, 17.85]^2, selected from
10^6 support points, sinusoidal bumps); per-scan recursive_update with a
20k-point scan inside a 2.5 m footprint (run with TLG_TRACE=1 for stages)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_26222_b200 import terrain as T  # noqa: E402


def bumps(x, y):
    return 0.05 * np.sin(2 * np.pi * x / 1.5) * np.sin(2 * np.pi * y / 1.5)


def main():
    rng = np.random.default_rng(4)
    side = 17.85
    sup = rng.uniform(0.0, side, size=(1_000_000, 2))
    cs = T.select_centers(T.TerrainObservation(sup, bumps(sup[:, 0], sup[:, 1])),
                          T.Rect((0.0, 0.0), (side, side)), 0.07, 0.12, 3)
    kernel = T.KernelParams()
    kernel.finalize()
    model = T.TerrainModel(kernel, cs)
    print(f"M = {model.num_centers()}", flush=True)

    def scan(cx, cy, m=20000):
        r = 2.5 * np.sqrt(rng.uniform(0, 1, m))
        a = rng.uniform(0, 2 * np.pi, m)
        clean = np.stack([cx + r * np.cos(a), cy + r * np.sin(a)], 1)
        noisy = clean + rng.normal(0.0, 0.02, size=(m, 2))
        return T.TerrainObservation(np.ascontiguousarray(noisy), bumps(clean[:, 0], clean[:, 1]))

    for k in range(8):
        s = scan(4.0 + 0.5 * k, 8.0 + 0.3 * k)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = model.recursive_update(s, False)
        dt = (time.perf_counter() - t0) * 1e3
        print(f"scan {k}: {dt:.3f} ms solver={rep.solver} n_active={rep.active_centers} "
              f"blocks={rep.active_blocks} rejected={rep.rejected}", flush=True)


if __name__ == "__main__":
    main()
