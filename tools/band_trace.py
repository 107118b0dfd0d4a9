"""Critical-path stamps of the forward dataflow band solve (diagnostics build
with -DTLG_FLOW_TRACE, dense.cu): for blocks 300..363 of the C5 batch fit,
per block, forward and backward (microseconds relative to the previous
block's release): staged +
older tiles done, critical flag observed, right-hand side reduced, diagonal
steps done, released."""
import ctypes as C
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
assert lib.tlg_debug_band_trace(buf) == 0
ab = np.array(buf, dtype=np.float64).reshape(2, 64, 8)
for name, a in (("forward", ab[0]), ("backward", ab[1])):
    print(name, "blk   start  ready  seen   rhs   diag  released   (us after the previous release)")
    for k in range(1, 64):
        p = a[k - 1, 5]
        r = (a[k, :8] - p) / 1e3 if name == "backward" else (a[k, :6] - p) / 1e3
        print(f"{300 + k:4d} " + " ".join(f"{v:6.2f}" for v in r))
