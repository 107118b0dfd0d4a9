"""RBFT snapshot save / load timing (C3-size model, 4,096 centres)."""
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2509_26222_b200 import terrain as T  # noqa: E402

k = T.KernelParams()
k.finalize()
roi = T.Rect((0.0, 0.0), (4.41, 4.41))
g = T.TerrainModel(k, T.CenterSet(np.zeros((0, 2)), 0.07, 0.12, 3, roi))
rng = np.random.default_rng(3)
xy = rng.uniform(0, 4.41, (20000, 2))
g.recursive_update(T.TerrainObservation(xy, bench.staircase(xy[:, 0])))
with tempfile.TemporaryDirectory() as td:
    p = str(Path(td) / "m.rbft")
    for i in range(3):
        t0 = time.perf_counter()
        g.save(p)
        t1 = time.perf_counter()
        h = T.TerrainModel.load(p)
        t2 = time.perf_counter()
        print(f"save {(t1 - t0) * 1e3:.1f} ms load {(t2 - t1) * 1e3:.1f} ms "
              f"({Path(p).stat().st_size} bytes, {h.num_centers()} centres)", flush=True)
