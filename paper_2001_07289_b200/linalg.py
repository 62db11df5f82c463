"""Sparse symmetric storage, error classes and the host-side tridiagonal eigensolver.

Mirrors ``bddcso.linalg`` (reference ``pkg/src/bddcso/linalg.py``):

* ``NotSpdError`` / ``UnderconstrainedError``   ↔ linalg.py:16-21
* ``SparseSym``                                  ↔ linalg.py:24-90 (upper-triangle CSR, lazy mirror)
* ``spd_factor`` / ``spd_solve``                 ↔ linalg.py:117-142 — here a dense FP64 Cholesky
  on the GPU (``csrc/dense_f64.cu``), not SuperLU
* ``saddle_factor`` / ``saddle_solve``           ↔ linalg.py:145-212 — GPU augmented-Lagrangian
  Cholesky that reproduces the reference's 1/s scaling of (g, λ)
* ``dense_sym_eig`` / ``tridiag_eig``            ↔ linalg.py:215-237 (LAPACK on the host; tiny)
"""

from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.sparse as sp


class NotSpdError(ValueError):
    """A factorization met a nonpositive pivot (linalg.py:16)."""


class UnderconstrainedError(ValueError):
    """A saddle system is singular: floating subdomain underconstrained (linalg.py:20)."""


class SparseSym:
    """Symmetric sparse matrix stored once in its upper triangle (linalg.py:24-90)."""

    def __init__(self, upper: sp.csr_matrix):
        n, m = upper.shape
        if n != m:
            raise ValueError("matrix must be square")
        coo = upper.tocoo()
        if np.any(coo.row > coo.col):
            raise ValueError("upper-triangle storage contains lower entries")
        self.n = n
        self.upper = upper.tocsr()
        self.upper.sum_duplicates()
        self._full = None

    @classmethod
    def from_upper_triplets(cls, n, rows, cols, data) -> "SparseSym":
        return cls(sp.coo_matrix((data, (rows, cols)), shape=(n, n)).tocsr())

    @classmethod
    def from_dense(cls, dense) -> "SparseSym":
        dense = np.asarray(dense, dtype=float)
        if not np.array_equal(dense, dense.T):
            raise ValueError("dense input is not symmetric")
        return cls(sp.triu(sp.csr_matrix(dense), format="csr"))

    @property
    def shape(self):
        return (self.n, self.n)

    @property
    def nnz(self) -> int:
        return self.upper.nnz

    def diagonal(self) -> np.ndarray:
        return self.upper.diagonal()

    def tocsr(self) -> sp.csr_matrix:
        if self._full is None:
            strict = sp.triu(self.upper, k=1)
            self._full = (self.upper + strict.T).tocsr()
        return self._full

    def tocsc(self) -> sp.csc_matrix:
        return self.tocsr().tocsc()

    def todense(self) -> np.ndarray:
        return self.tocsr().toarray()

    def matvec(self, x: np.ndarray) -> np.ndarray:
        return self.tocsr() @ x

    def __matmul__(self, x):
        return self.matvec(x)

    def restrict(self, idx: np.ndarray) -> "SparseSym":
        idx = np.asarray(idx)
        sub = self.tocsr()[idx][:, idx]
        return SparseSym(sp.triu(sub, format="csr"))

    def scaled(self, factor: float) -> "SparseSym":
        return SparseSym(self.upper * factor)


def dense_sym_eig(matrix) -> np.ndarray:
    """Eigenvalues (ascending) of a dense symmetric matrix (linalg.py:215-223)."""
    M = np.asarray(matrix, dtype=float)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("matrix must be square")
    scale = np.abs(M).max() if M.size else 1.0
    scale = scale or 1.0
    if np.abs(M - M.T).max(initial=0.0) > 1e-12 * scale:
        raise ValueError("matrix is not symmetric")
    return np.linalg.eigvalsh(0.5 * (M + M.T))


def tridiag_eig(alphas, betas):
    """Extreme eigenvalues (min, max) of a symmetric tridiagonal matrix (linalg.py:226-237)."""
    d = np.asarray(alphas, dtype=float)
    e = np.asarray(betas, dtype=float)
    if d.size == 0:
        raise ValueError("empty tridiagonal matrix")
    if e.size != d.size - 1:
        raise ValueError("off-diagonal length must be len(diagonal) - 1")
    if d.size == 1:
        return float(d[0]), float(d[0])
    vals = scipy.linalg.eigvalsh_tridiagonal(d, e)
    return float(vals[0]), float(vals[-1])


def __getattr__(name):
    # device-backed factorizations live in _dense.py (they need the CUDA library)
    if name in ("spd_factor", "spd_solve", "saddle_factor", "saddle_solve",
                "SpdFactorization", "SaddleFactorization"):
        from . import _dense

        return getattr(_dense, name)
    raise AttributeError(name)
