"""Headline step overhead: CUDA-event time per LM evaluation through the
Python wrapper vs a direct C-ABI call with prebuilt arguments vs the kernel."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2509_26222_b200 import _abi  # noqa: E402
from paper_2509_26222_b200 import kinematics as kin  # noqa: E402
from paper_2509_26222_b200 import terrain as T  # noqa: E402

model, kernel, cs, w, R, tv, h = bench.build_c5(0, 10_000_000, 1000, torch)
n = 10_000_000
rows = {"r": torch.empty(n, dtype=torch.float64, device="cuda"),
        "J": torch.empty(6 * n, dtype=torch.float64, device="cuda"),
        "valid": torch.empty(n, dtype=torch.uint8, device="cuda")}
R0 = bench.so3_exp(np.array(bench.POSE_W) + np.array([0.004, -0.003, 0.01]))
scan = kin.Scan(model, R0, tv + np.array([0.03, -0.02, 0.01]), h)
lib = _abi.load()
Rm = np.ascontiguousarray(np.asarray(R).reshape(9))
tvv = np.ascontiguousarray(tv)
ne = _abi.NormalEqC()
args = (model.handle, scan.handle, Rm.ctypes.data, tvv.ctypes.data, 0.0, 1.0, 0.05,
        rows["r"].data_ptr(), rows["J"].data_ptr(), rows["valid"].data_ptr(), None,
        _abi.TLG_DEVICE, C.byref(ne))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for label, f in (("wrapper", lambda: scan.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rows)),
                 ("direct", lambda: lib.tlg_scan_manifold_rows(*args))):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / 50:.4f} ms/step", flush=True)
ctx = T.Context.default(0)
lib.tlg_ctx_set_profiling(ctx.handle, 1)
for _ in range(20):
    lib.tlg_scan_manifold_rows(*args)
ms, cnt = C.c_double(), C.c_uint64()
lib.tlg_ctx_kernel_stats(ctx.handle, 0, C.byref(ms), C.byref(cnt))
print(f"k_manifold {ms.value / cnt.value:.4f} ms", flush=True)
