import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import bench
from paper_2509_26222_b200 import terrain as T
rng = np.random.default_rng(4)
side = 17.85
sup = rng.uniform(0.0, side, size=(1_000_000, 2))
cs = T.select_centers(T.TerrainObservation(sup, bench.terrain_c5(sup[:, 0], sup[:, 1], np)), T.Rect((0.0, 0.0), (side, side)), 0.07, 0.12, 3)
k = T.KernelParams(); k.finalize()
obs = T.TerrainObservation(sup, bench.terrain_c5(sup[:, 0], sup[:, 1], np))
for i in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    m = T.TerrainModel(k, cs)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    T.fit_batch_ridge(k, cs, obs)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"model ctor {1e3*(t1-t0):.1f} ms, fit_batch_ridge {1e3*(t2-t1):.1f} ms", flush=True)
