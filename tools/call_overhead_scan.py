"""Host overhead of Scan.manifold_rows per call: wall time per call on the C5
scan (10^7 points) and on a 32-point scan, plus a cProfile of the small call."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_26222_b200 import kinematics as kin  # noqa: E402


def rows_for(n):
    return {"r": torch.empty(n, dtype=torch.float64, device="cuda"),
            "J": torch.empty(6 * n, dtype=torch.float64, device="cuda"),
            "valid": torch.empty(n, dtype=torch.uint8, device="cuda")}


def per_call(scan, rows, R, tv, reps):
    for _ in range(5):
        scan.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rows)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        scan.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rows)
    return (time.perf_counter() - t0) / reps * 1e6


def main():
    model, kernel, cs, w, R, tv, h = bench.build_c5(0, 10_000_000, 7, torch)
    big = kin.Scan(model, R, tv, h)
    print(f"C5 call: {per_call(big, rows_for(big.n), R, tv, 200):.1f} us wall")
    small_h = tuple(a[:32].contiguous() for a in h)
    small = kin.Scan(model, R, tv, small_h)
    rs = rows_for(small.n)
    print(f"32-point call: {per_call(small, rs, R, tv, 500):.1f} us wall")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(500):
        small.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rs)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(8)


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def bench_like():
    """The bench's timed loop (perturbed binning pose, CUDA events around the
    steps) with and without the library's per-call kernel profiling."""
    import numpy as np
    from paper_2509_26222_b200 import _abi
    from paper_2509_26222_b200 import terrain as T
    ctx = T.Context.default(0)
    model, kernel, cs, w, R, tv, h = bench.build_c5(0, 10_000_000, 1000, torch)
    rows = rows_for(10_000_000)
    R0 = bench.so3_exp(np.array(bench.POSE_W) + np.array([0.004, -0.003, 0.01]))
    kin.Scan(model, R0, tv, h)
    scan = kin.Scan(model, R0, tv + np.array([0.03, -0.02, 0.01]), h)
    lib = _abi.load()
    for prof in (0, 1, 0, 1):
        lib.tlg_ctx_set_profiling(ctx.handle, prof)
        for _ in range(5):
            scan.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rows)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            scan.manifold_rows(R, tv, 0.0, 1.0, 0.05, out=rows)
        e1.record()
        torch.cuda.synchronize()
        print(f"profiling={prof}: {e0.elapsed_time(e1) / 20:.4f} ms/step")
    lib.tlg_ctx_set_profiling(ctx.handle, 0)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "--bench-like":
    bench_like()
