"""C1 per-stage timing (BASELINE configs[0]): M = 256 lattice on [0, 1.05]^2,
one 20k-point scan; run with TLG_TRACE=1 for the update's stages."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_26222_b200 import terrain as T  # noqa: E402


def main():
    xy, z = bench.c1_inputs_np()
    roi = T.Rect((0.0, 0.0), (1.05, 1.05))
    obs = T.TerrainObservation(xy, z)
    k = T.KernelParams()
    k.finalize()
    cs = T.select_centers(obs, roi, 0.07, 0.12, 3)
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m = T.TerrainModel(k, cs)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rep = m.recursive_update(obs, False)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"iter {it}: model create {1e3 * (t1 - t0):.3f} ms, update {1e3 * (t2 - t1):.3f} ms "
              f"({rep.solver}, n={rep.active_centers})", flush=True)


if __name__ == "__main__":
    main()
