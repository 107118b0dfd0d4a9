"""Fixed per-call overhead of tlg_scan_manifold_rows (tiny scan) and of the
bench step at 10^7 points (wall clock vs kernel time)."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_26222_b200 import kinematics as kin  # noqa: E402

for n in (1024, 10_000_000):  # noqa
    model, kernel, cs, w, R, tv, h = bench.build_c5(0, n, 7, torch)
    scan = kin.Scan(model, R, tv, h)
    rows = {"r": torch.empty(n, dtype=torch.float64, device="cuda"),
            "J": torch.empty(6 * n, dtype=torch.float64, device="cuda"),
            "valid": torch.empty(n, dtype=torch.uint8, device="cuda")}
    for _ in range(5):
        scan.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rows)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        scan.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rows)
    dt = (time.perf_counter() - t0) / 50 * 1e6
    print(f"n={n}: {dt:.1f} us per call (wall)", flush=True)

# raw ctypes call (no Python wrapper work) on the last scan
import ctypes as C  # noqa: E402
from paper_2509_26222_b200 import _abi  # noqa: E402
lib = _abi.load()
Rm = np.ascontiguousarray(np.asarray(R, dtype=np.float64).reshape(9))
tv2 = np.ascontiguousarray(np.asarray(tv, dtype=np.float64).reshape(3))
ne = kin.NormalEqC()
args = (model.handle, scan.handle, Rm.ctypes.data_as(C.c_void_p), tv2.ctypes.data_as(C.c_void_p),
        0.0, 1.0, 0.05, C.c_void_p(rows["r"].data_ptr()), C.c_void_p(rows["J"].data_ptr()),
        C.c_void_p(rows["valid"].data_ptr()), None, _abi.TLG_DEVICE, C.byref(ne))
for nn in (1024,):
    pass
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    lib.tlg_scan_manifold_rows(*args)
print(f"raw ctypes (n=1e7 scan): {(time.perf_counter() - t0) / 50 * 1e6:.1f} us per call", flush=True)
