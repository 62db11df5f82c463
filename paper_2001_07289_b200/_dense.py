"""Dense FP64 factorizations on the GPU with the reference's ``linalg`` API (linalg.py:101-212).

The reference factors with SuperLU (SPD: symmetric mode, MMD_AT_PLUS_A, no pivoting;
KKT: LU of [[A, sC^T], [sC, 0]] with s = mean |diag A|). Here the matrices are densified
and factored by this library's Cholesky (csrc/dense_f64.cu, C ABI ``bddc_dense_potrf`` /
``bddc_dense_trsm``); the KKT system is solved by the augmented-Lagrangian form the device
operator uses (K = A + s C^T C, S = C K^{-1} C^T), reproducing the reference's scaling
quirk: ``solve`` returns u with C u = g / s^2 and lam = lambda / s^2 (linalg.py:158-172, 208).

Errors keep the reference's classes and messages: NotSpdError on a nonpositive pivot of an
SPD factorization, UnderconstrainedError when K or S is not positive definite.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import scipy.sparse as sp

from . import _capi
from .linalg import NotSpdError, SparseSym, UnderconstrainedError

_NO_FAIL = -1  # bddc_dense_potrf: -1 = factored, else first failing pivot


def _dense(matrix) -> np.ndarray:
    if isinstance(matrix, SparseSym):
        return np.asarray(matrix.todense(), dtype=float)
    if sp.issparse(matrix):
        return matrix.toarray().astype(float)
    return np.asarray(matrix, dtype=float)


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("dense factorizations need a CUDA GPU (no CPU fallback)")
    return torch


def _colmajor(torch, M: np.ndarray, ld: int):
    """Device column-major copy with even leading dimension: tensor[col, row]."""
    n_rows, n_cols = M.shape
    T = torch.zeros((max(n_cols, 1), ld), dtype=torch.float64, device="cuda")
    if n_rows and n_cols:
        T[:n_cols, :n_rows] = torch.from_numpy(np.ascontiguousarray(M.T)).cuda()
    return T


def _potrf(torch, T, n: int, ld: int) -> int:
    lib = _capi.load()
    info = (C.c_int * 1)()
    stream = torch.cuda.current_stream().cuda_stream
    rc = lib.bddc_dense_potrf(C.c_void_p(T.data_ptr()), n, ld, ld * n, 1, info, C.c_void_p(stream))
    if rc:
        raise RuntimeError(f"bddc_dense_potrf failed ({rc})")
    return int(info[0])


def _trsm(torch, kind: int, L, n: int, ld: int, B, nrhs: int, ldb: int):
    lib = _capi.load()
    stream = torch.cuda.current_stream().cuda_stream
    rc = lib.bddc_dense_trsm(kind, C.c_void_p(L.data_ptr()), n, ld, ld * n, C.c_void_p(B.data_ptr()),
                             nrhs, ldb, ldb * nrhs, 1, C.c_void_p(stream))
    if rc:
        raise RuntimeError(f"bddc_dense_trsm failed ({rc})")


def _gemm(torch, tA: bool, tB: bool, M: int, N: int, K: int, alpha: float, A, lda: int, B, ldb: int,
          beta: float, Cm, ldc: int):
    """C = alpha op(A) op(B) + beta C on column-major device tensors (this library's DMMA GEMM)."""
    lib = _capi.load()
    stream = torch.cuda.current_stream().cuda_stream
    rc = lib.bddc_dense_gemm(int(tA), int(tB), M, N, K, float(alpha), C.c_void_p(A.data_ptr()), lda, 0,
                             C.c_void_p(B.data_ptr()), ldb, 0, float(beta), C.c_void_p(Cm.data_ptr()),
                             ldc, 0, 1, C.c_void_p(stream))
    if rc:
        raise RuntimeError(f"bddc_dense_gemm failed ({rc})")


class SpdFactorization:
    """Cholesky factor of an SPD matrix on the GPU (linalg.py:101-114)."""

    def __init__(self, L, n: int, ld: int):
        self._L, self.n, self._ld = L, n, ld
        self.permutation = np.arange(n)  # dense factor: identity ordering

    def _solve_dev(self, torch, B, nrhs):
        _trsm(torch, 0, self._L, self.n, self._ld, B, nrhs, self._ld)  # L y = b
        _trsm(torch, 1, self._L, self.n, self._ld, B, nrhs, self._ld)  # L^T x = y

    def solve(self, rhs: np.ndarray) -> np.ndarray:
        torch = _torch()
        b = np.asarray(rhs, dtype=float)
        if b.shape[0] != self.n:
            raise ValueError("right-hand side dimensions do not match factorization")
        B2 = b.reshape(self.n, -1)
        nrhs = B2.shape[1]
        B = _colmajor(torch, B2, self._ld)
        self._solve_dev(torch, B, nrhs)
        return B[:nrhs, :self.n].T.cpu().numpy().reshape(b.shape)


def spd_factor(matrix) -> SpdFactorization:
    """Factor a symmetric positive definite matrix for repeated solves (linalg.py:117-138)."""
    torch = _torch()
    A = _dense(matrix)
    n = A.shape[0]
    if n == 0:
        raise ValueError("cannot factor an empty matrix")
    ld = n + (n & 1)
    T = _colmajor(torch, A, ld)
    bad = _potrf(torch, T, n, ld)
    if bad != _NO_FAIL:
        raise NotSpdError(f"matrix not SPD: nonpositive pivot at index {bad}")
    return SpdFactorization(T, n, ld)


def spd_solve(fact: SpdFactorization, rhs: np.ndarray) -> np.ndarray:
    return fact.solve(rhs)


class SaddleFactorization:
    """[[A, C^T], [C, 0]] through K = A + s C^T C and S = C K^{-1} C^T (linalg.py:145-172)."""

    def __init__(self, K: SpdFactorization, Cd: np.ndarray, s: float, S: SpdFactorization | None,
                 G):
        self._K, self._C, self._s, self._S, self._G = K, Cd, s, S, G
        self.n, self.m = K.n, Cd.shape[0]

    def solve(self, f: np.ndarray, g: np.ndarray):
        """(u, lam) with C u = g / s^2 and A u + C^T (s^2 lam) = f (the reference's scaling)."""
        torch = _torch()
        f = np.asarray(f, dtype=float)
        g = np.asarray(g, dtype=float)
        if f.shape[0] != self.n or g.shape[0] != self.m:
            raise ValueError("right-hand side dimensions do not match factorization")
        if self.m == 0:
            return self._K.solve(f), np.zeros((0,) + f.shape[1:])
        s = self._s
        F = f.reshape(self.n, -1)
        gp = g.reshape(self.m, -1) / (s * s)  # the constraint the reference enforces
        nrhs = F.shape[1]
        Cd = self._C
        # h = L^{-1} (f + s C^T g'), lambda = S^{-1} (G^T h - g'), u = L^{-T} (h - G lambda)
        H = _colmajor(torch, F + s * (Cd.T @ gp), self._K._ld)
        _trsm(torch, 0, self._K._L, self.n, self._K._ld, H, nrhs, self._K._ld)
        G = self._G  # column-major n x m: L^{-1} C^T
        ld, m, n = self._K._ld, self.m, self.n
        ldm = m + (m & 1)
        R = torch.zeros((nrhs, ldm), dtype=torch.float64, device="cuda")
        _gemm(torch, True, False, m, nrhs, n, 1.0, G, ld, H, ld, 0.0, R, ldm)  # G^T h
        rhs_l = R[:, :m].T.cpu().numpy() - gp
        lam_true = self._S.solve(rhs_l.reshape((self.m,) + g.shape[1:])).reshape(self.m, -1)
        Lt = _colmajor(torch, lam_true, ldm)
        _gemm(torch, False, False, n, nrhs, m, -1.0, G, ld, Lt, ldm, 1.0, H, ld)  # h - G lambda
        _trsm(torch, 1, self._K._L, self.n, self._K._ld, H, nrhs, self._K._ld)
        u = H[:nrhs, :self.n].T.cpu().numpy().reshape(f.shape)
        lam = (lam_true / (s * s)).reshape((self.m,) + g.shape[1:])
        return u, lam


def saddle_factor(A, C) -> SaddleFactorization:
    """Factor the KKT system of a semidefinite A with constraints C (linalg.py:175-208)."""
    torch = _torch()
    Ad = _dense(A)
    n = Ad.shape[0]
    Cd = _dense(C) if C is not None else np.zeros((0, n))
    if Cd.ndim != 2 or Cd.shape[1] != n:
        raise ValueError("constraint matrix column count does not match A")
    m = Cd.shape[0]
    msg = ("saddle system numerically singular (floating subdomain underconstrained "
           "or rank-deficient constraints)")
    s = (float(np.mean(np.abs(np.diag(Ad)))) or 1.0) if m else 1.0
    try:
        K = spd_factor(Ad + s * (Cd.T @ Cd) if m else Ad)
    except NotSpdError as err:
        raise UnderconstrainedError(msg) from err
    if m == 0:
        return SaddleFactorization(K, Cd, 1.0, None, None)
    G = _colmajor(torch, Cd.T, K._ld)  # C^T, n x m
    _trsm(torch, 0, K._L, n, K._ld, G, m, K._ld)
    ldm = m + (m & 1)
    Sd = torch.zeros((m, ldm), dtype=torch.float64, device="cuda")
    _gemm(torch, True, False, m, m, n, 1.0, G, K._ld, G, K._ld, 0.0, Sd, ldm)  # S = G^T G
    S = Sd[:, :m].cpu().numpy()
    S = 0.5 * (S + S.T)
    try:
        Sf = spd_factor(S)
    except NotSpdError as err:
        raise UnderconstrainedError(msg) from err
    return SaddleFactorization(K, Cd, s, Sf, G)


def saddle_solve(fact: SaddleFactorization, f: np.ndarray, g: np.ndarray):
    return fact.solve(f, g)


__all__ = ["SpdFactorization", "SaddleFactorization", "spd_factor", "spd_solve", "saddle_factor",
           "saddle_solve"]
