"""Times k_manifold (scan-binned C5 workload) with the library's CUDA-event
kernel profiling; prints one line per run. Used for A/B kernel variants via
TLG_LIB_OVERRIDE."""
import argparse
import ctypes as C
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_26222_b200 import _abi  # noqa: E402
from paper_2509_26222_b200 import kinematics as kin  # noqa: E402
from paper_2509_26222_b200 import terrain as T  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--points", type=int, default=10_000_000)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--unbinned", action="store_true")
    ap.add_argument("--eval", action="store_true")
    ap.add_argument("--generic", action="store_true",
                    help="jitter the centres off the lattice (generic sweep)")
    a = ap.parse_args()
    model, kernel, cs, w, R, tv, h = bench.build_c5(0, a.points, 7, torch)
    if a.generic:
        import numpy as np
        rng = np.random.default_rng(3)
        c = cs.centers + rng.uniform(-0.005, 0.005, cs.centers.shape)
        cs = T.CenterSet(c, cs.mesh_resolution, cs.accept_radius, cs.accept_count, cs.roi)
        model = T.TerrainModel(kernel, cs)
        model.set_weights(w)
        print("sweep kind", model.sweep(), flush=True)
    n = a.points
    rows = {"r": torch.empty(n, dtype=torch.float64, device="cuda"),
            "J": torch.empty(6 * n, dtype=torch.float64, device="cuda"),
            "valid": torch.empty(n, dtype=torch.uint8, device="cuda")}
    scan = None if a.unbinned else kin.Scan(model, R, tv, h)

    def run():
        if scan is None:
            return kin.manifold_rows(model, R, tv, h, 0.0, 1.0, 0.05, out=rows)[1]
        return scan.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rows)[1]

    for _ in range(3):
        run()
    lib = _abi.load()
    ctx = T.Context.default(0)
    lib.tlg_ctx_set_profiling(ctx.handle, 1)
    for _ in range(a.iters):
        ne = run()
    ms, cnt = C.c_double(), C.c_uint64()
    lib.tlg_ctx_kernel_stats(ctx.handle, 0, C.byref(ms), C.byref(cnt))
    k = ms.value / cnt.value
    print(f"{os.environ.get('TLG_LIB_OVERRIDE', 'default')}: k_manifold {k:.4f} ms  "
          f"{n / k / 1e6:.3f} Gpts/s  {81 * n / (k * 1e-3) / 1e9:.1f} GB/s  cost={ne.cost:.6g}",
          flush=True)
    if a.eval:
        # K3 batch predict (height + gradient + supported) on the same points
        # in scan order (binned) and in generation order
        xy = torch.stack([h[0], h[1]], 1).contiguous()
        key = torch.floor(xy[:, 0] / 0.07) * 1e6 + torch.floor(xy[:, 1] / 0.07)
        binned = xy[torch.argsort(key)].contiguous()
        for exact in (False, True):
            model.set_exact_cutoff(exact)
            for label, q in (("random order", xy), ("binned", binned)):
                model.predict(q)
                lib.tlg_ctx_set_profiling(ctx.handle, 1)
                for _ in range(a.iters):
                    model.predict(q)
                lib.tlg_ctx_kernel_stats(ctx.handle, 1, C.byref(ms), C.byref(cnt))
                k = ms.value / cnt.value
                print(f"k_eval ({label}, sweep {model.sweep()[0]}): {k:.4f} ms  "
                      f"{n / k / 1e6:.3f} Gpts/s  {41 * n / (k * 1e-3) / 1e9:.1f} GB/s", flush=True)
        model.set_exact_cutoff(False)


if __name__ == "__main__":
    main()
