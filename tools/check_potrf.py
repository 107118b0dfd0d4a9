"""Numerics + timing of the device Cholesky (tlg_debug_potrf / dense bench)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2509_26222_b200 import _abi  # noqa: E402
from paper_2509_26222_b200 import terrain as T  # noqa: E402


def potrf(A, tile=0):
    n = A.shape[0]
    A = np.asfortranarray(A, dtype=np.float64)
    L = np.zeros((n, n), order="F")
    X = np.zeros((n, n), order="F")
    _abi.check(_abi.load_diag().tlg_diag_potrf(T.Context.default().handle, n, A.ctypes.data, tile, 0,
                                           L.ctypes.data, X.ctypes.data))
    return L, X


if __name__ == "__main__":
    rng = np.random.default_rng(0)
    for n in (1, 5, 31, 32, 33, 64, 100, 400, 1000, 1100):
        G = rng.standard_normal((n, n))
        A = G @ G.T + n * np.eye(n)
        for tile in (32, 64):
            L, X = potrf(A, tile)
            e1 = np.abs(L @ L.T - A).max() / np.abs(A).max()
            e2 = np.abs(X @ L - np.eye(n)).max()
            print(f"n={n:5d} tile={tile}: |LL^T-A|/|A|={e1:.2e} |XL-I|={e2:.2e}")
    from dense_bench import run
    for n in (64, 128, 256, 400, 1024):
        print(f"n={n}: potrf {run(0, n, 0) * 1e3:.1f} us, potrf+X {run(5, n, 0) * 1e3:.1f} us, "
              f"potrf64 {run(6, n, 0) * 1e3:.1f} us")
