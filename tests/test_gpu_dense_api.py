"""Reference linalg API on the GPU dense kernels (_dense.py, linalg.py:101-212): SPD solves,
the KKT solve with the reference's 1/s scaling quirk, and the error classes/messages."""
import numpy as np
import pytest

import paper_2001_07289_b200 as P

pytestmark = pytest.mark.gpu


def _laplacian_1d(n):
    A = np.zeros((n, n))
    for i in range(n - 1):
        A[i, i] += 1.0
        A[i + 1, i + 1] += 1.0
        A[i, i + 1] -= 1.0
        A[i + 1, i] -= 1.0
    return A  # floating: kernel = constants


def test_spd_factor_solve(cuda_ok):
    rng = np.random.default_rng(0)
    for n in (1, 7, 37, 64, 130):
        M = rng.standard_normal((n, n))
        A = M @ M.T + n * np.eye(n)
        f = P.spd_factor(A)
        b = rng.standard_normal(n)
        B = rng.standard_normal((n, 3))
        assert np.allclose(f.solve(b), np.linalg.solve(A, b), rtol=1e-12, atol=1e-12)
        assert np.allclose(P.spd_solve(f, B), np.linalg.solve(A, B), rtol=1e-12, atol=1e-12)


def test_spd_factor_not_spd(cuda_ok):
    A = np.diag([4.0, 1.0, -2.0, 3.0])
    with pytest.raises(P.NotSpdError, match="nonpositive pivot at index 2"):
        P.spd_factor(A)


def test_saddle_matches_reference_kkt(cuda_ok):
    n = 20
    A = _laplacian_1d(n) * 3.0 + np.diag(np.r_[np.zeros(n - 1), 0.0])
    C = np.zeros((2, n))
    C[0, :] = 1.0 / n   # mean (edge-like) constraint
    C[1, 5] = 1.0       # vertex constraint
    rng = np.random.default_rng(1)
    f = rng.standard_normal(n)
    g = rng.standard_normal(2)
    fac = P.saddle_factor(A, C)
    u, lam = P.saddle_solve(fac, f, g)
    # the reference: LU of [[A, sC^T], [sC, 0]] with rhs [f; g/s], lam = sol[n:] / s
    s = float(np.mean(np.abs(np.diag(A))))
    K = np.block([[A, s * C.T], [s * C, np.zeros((2, 2))]])
    sol = np.linalg.solve(K, np.r_[f, g / s])
    assert np.allclose(u, sol[:n], rtol=1e-10, atol=1e-10)
    assert np.allclose(lam, sol[n:] / s, rtol=1e-10, atol=1e-10)
    # multi-RHS (the coarse-basis solve g = I)
    U, L = fac.solve(np.zeros((n, 2)), np.eye(2))
    sol2 = np.linalg.solve(K, np.r_[np.zeros((n, 2)), np.eye(2) / s])
    assert np.allclose(U, sol2[:n], rtol=1e-10, atol=1e-10)


def test_saddle_underconstrained(cuda_ok):
    A = _laplacian_1d(8)
    with pytest.raises(P.UnderconstrainedError):
        P.saddle_factor(A, np.zeros((0, 8)))
