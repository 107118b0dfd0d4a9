"""Small driver for ncu captures of the hot kernels (one GPU).

Runs the C5 model with --points lever arms: a few scan-binned manifold-row
evaluations (k_manifold) and one batched height/gradient eval (k_eval).
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_26222_b200 import kinematics as kin  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=2_000_000)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--unbinned", action="store_true")
    a = ap.parse_args()
    model, kernel, cs, w, R, tv, h = bench.build_c5(0, a.points, 7, torch)
    n = a.points
    rows = {"r": torch.empty(n, dtype=torch.float64, device="cuda"),
            "J": torch.empty(6 * n, dtype=torch.float64, device="cuda"),
            "valid": torch.empty(n, dtype=torch.uint8, device="cuda")}
    if a.unbinned:
        for _ in range(a.iters):
            _, ne = kin.manifold_rows(model, R, tv, h, 0.0, 1.0, 0.05, out=rows)
    else:
        scan = kin.Scan(model, R, tv, h)
        for _ in range(a.iters):
            _, ne = scan.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rows)
    xy = torch.stack([h[0], h[1]], 1)
    model.predict(xy)
    torch.cuda.synchronize()
    print("ok", ne.valid, ne.cost)


if __name__ == "__main__":
    main()
