"""C5 batch-system assembly alone (10^7 points, 99,856 lattice centres),
for ncu launch lists / captures of the lattice element assembly
(assemble.cu) and, with --csr, the row-wise CSR Gram."""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2509_26222_b200 import _abi  # noqa: E402
from paper_2509_26222_b200 import terrain as T  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=10_000_000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--csr", action="store_true")
    a = ap.parse_args()
    side = bench.ROI_C5[1][0]
    nodes = np.arange(int(round(side / bench.RES)) + 1) * bench.RES
    gx, gy = np.meshgrid(nodes, nodes, indexing="ij")
    cs = T.CenterSet(np.stack([gx.ravel(), gy.ravel()], 1), bench.RES, bench.R_A, bench.COUNT,
                     T.Rect(*bench.ROI_C5))
    k = T.KernelParams()
    k.finalize()
    model = T.TerrainModel(k, cs)
    _abi.check(_abi.load_diag().tlg_diag_set_batch_gram(model.handle, 1 if a.csr else 0))
    n, ld, el = model.batch_system()
    g = torch.Generator(device="cuda").manual_seed(11)
    xy = torch.rand((a.points, 2), generator=g, device="cuda", dtype=torch.float64) * side
    z = bench.terrain_c5(xy[:, 0], xy[:, 1], torch)
    H = torch.empty(el, dtype=torch.float64, device="cuda")
    b = torch.empty(n, dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r in range(a.reps):
        torch.cuda.synchronize()
        e0.record()
        model.batch_assemble(xy, z, H, b, add_lambda=True)
        e1.record()
        torch.cuda.synchronize()
        print(f"assemble {'csr' if a.csr else 'lattice'} rep {r}: {e0.elapsed_time(e1):.3f} ms",
              flush=True)


if __name__ == "__main__":
    main()
