"""C3 update latency breakdown: M = 4096 lattice model, per-scan
recursive_update at m = 400 and 20,000 (run with TLG_TRACE=1 for stages)."""
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
    roi = T.Rect((0.0, 0.0), (4.41, 4.41))
    kernel = T.KernelParams()
    kernel.finalize()
    model = T.TerrainModel(kernel, T.CenterSet(np.zeros((0, 2)), 0.07, 0.12, 3, roi))
    rng = np.random.default_rng(3)

    def scan(m):
        clean = rng.uniform(0.0, 4.41, size=(m, 2))
        noisy = clean + rng.normal(0.0, 0.1, size=(m, 2))
        return T.TerrainObservation(np.ascontiguousarray(noisy), bench.staircase(clean[:, 0]))

    model.recursive_update(scan(20000))
    for m in [int(a) for a in (sys.argv[1:] or ["400", "20000"])]:
        for i in range(4):
            s = scan(m)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = model.recursive_update(s)
            dt = (time.perf_counter() - t0) * 1e3
            print(f"m={m} iter={i} {dt:.3f} ms solver={rep.solver} n={rep.active_centers}",
                  flush=True)


if __name__ == "__main__":
    main()
