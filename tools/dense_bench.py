"""Dense-solver microbenchmarks (tlg_debug_dense_bench) on one GPU."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2509_26222_b200 import _abi  # noqa: E402
from paper_2509_26222_b200 import terrain as T  # noqa: E402


def run(op, n, nrhs, reps=5):
    ms = C.c_double()
    _abi.check(_abi.load_diag().tlg_diag_dense_bench(T.Context.default().handle, op, n, nrhs, reps,
                                                  C.byref(ms)))
    return ms.value


if __name__ == "__main__":
    for reps in (1, 10):
        print(f"diag tile x{reps}: {run(3, 64, reps) * 1e3:.1f} us")
    for g in (1, 21, 148):
        print(f"grid.sync x100 with {g} CTAs: {run(4, g, 100) * 1e3 / 100:.2f} us each")
    for n in (64, 128, 256, 400, 1024):
        print(f"potrf n={n}: {run(0, n, 0) * 1e3:.1f} us")
    for n, r in ((400, 1), (400, 4096), (1024, 1)):
        print(f"trsm n={n} nrhs={r}: {run(1, n, r) * 1e3:.1f} us")
    for n, r in ((64, 64), (400, 400), (4096, 4096)):
        ms = run(2, n, r)
        print(f"gemm {n}x{r}x{n}: {ms * 1e3:.1f} us  {2.0 * n * n * r / ms / 1e9:.2f} TF/s")
