"""Critical-path stamps of the dataflow Cholesky (diagnostics build with
-DTLG_FLOW_TRACE: tools/build_variants.sh style, dense.cu): for columns
1000..1063 of the C5 batch fit, per column the diagonal task's claim / updates
done / Linv published and the first solve task's claim / updates done /
Linv observed / published, in microseconds relative to the diagonal claim."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import torch  # noqa: E402
from paper_2509_26222_b200 import _abi  # noqa: E402

out = bench.run_batch_fit_c5(torch, 0, 0, 1, 2_000_000)
lib = _abi.load()
buf = (C.c_ulonglong * (2 * 64 * 8))()
assert lib.tlg_debug_flow_trace(buf) == 0
a2 = np.array(buf, dtype=np.float64).reshape(2, 64, 8)
a, b = a2[0], a2[1]
t0 = a[:, 0:1]
rel = (a - t0) / 1e3
print("col  diag:upd  potrf:start potrf:end diag:pub | solve:upd solve:seen solve:pub | next diag pub")
for c in range(0, 63):
    nxt = (b[c + 1, 2] - b[c, 2]) / 1e3  # Linv published (warp 1, trace2 slot 2)
    ps, pe = (a[c, 7] - a[c, 0]) / 1e3, (b[c, 5] - a[c, 0]) / 1e3
    print(f"{1000 + c:5d} {rel[c, 1]:8.2f} {ps:8.2f} {pe:8.2f} {(b[c, 2] - a[c, 0]) / 1e3:8.2f} | {rel[c, 4]:9.2f} "
          f"{rel[c, 5]:9.2f} {rel[c, 6]:9.2f} | {nxt:8.2f}")
