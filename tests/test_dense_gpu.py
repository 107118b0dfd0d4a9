"""Device Cholesky + inverse factor (K7 dense layer) against numpy on random SPD
matrices, both tilings (32-wide register path, 64-wide tile path), ragged
sizes and the non-PD error path."""
import ctypes as C

import numpy as np
import pytest

from paper_2509_26222_b200 import _abi
from paper_2509_26222_b200 import terrain as T


def _potrf(A, tile, band=0):
    n = A.shape[0]
    A = np.asfortranarray(A, dtype=np.float64)
    L = np.zeros((n, n), order="F")
    X = np.zeros((n, n), order="F")
    _abi.check(_abi.load_diag().tlg_diag_potrf(T.Context.default().handle, n, A.ctypes.data, tile,
                                           band, L.ctypes.data, X.ctypes.data))
    return L, X


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 7, 32, 33, 95, 400, 1030])
@pytest.mark.parametrize("tile", [0, 32, 64])
def test_potrf_and_inverse(gpu_ctx, n, tile):
    rng = np.random.default_rng(n)
    G = rng.standard_normal((n, n))
    A = G @ G.T + n * np.eye(n)
    L, X = _potrf(A, tile)
    Lref = np.linalg.cholesky(A)
    assert np.abs(np.triu(L, 1)).max() == 0.0
    np.testing.assert_allclose(L, Lref, rtol=0, atol=1e-12 * np.abs(Lref).max())
    np.testing.assert_allclose(X @ L, np.eye(n), rtol=0, atol=1e-12)


@pytest.mark.gpu
# band 0: 32-wide diagonal blocks only (bwt = 0, no claim-order table); the
# others cover one-tile bands, ragged last tiles and the dense limit under
# the anti-diagonal task order with the interleaved L^-1 tasks
@pytest.mark.parametrize("n,band", [(300, 40), (1500, 200), (2000, 31), (700, 699), (200, 0), (95, 40), (1000, 5), (4100, 130)])
def test_potrf_banded(gpu_ctx, n, band):
    # block-banded SPD matrix (the information-form structure): the banded
    # factorisation must equal the dense one, and X = L^-1 stays exact
    rng = np.random.default_rng(band)
    G = rng.standard_normal((n, n))
    A = G @ G.T
    i, j = np.indices((n, n))
    A[np.abs(i - j) > band] = 0.0
    A += n * np.eye(n)
    L, X = _potrf(A, 0, band)
    Lref = np.linalg.cholesky(A)
    np.testing.assert_allclose(L, Lref, rtol=0, atol=1e-12 * np.abs(Lref).max())
    np.testing.assert_allclose(X @ L, np.eye(n), rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_potrf_not_pd(gpu_ctx):
    A = np.eye(40)
    A[17, 17] = -1.0
    with pytest.raises(_abi.DomainError):
        _potrf(A, 0)
