"""Preconditioned CG with a Lanczos condition estimate (reference krylov.py:31-104).

``pcg(apply_A, apply_B, b, tol, max_iters)`` keeps the reference signature. When
``apply_B`` is a device :class:`BddcOperator` (or its bound ``apply``) and ``apply_A`` is
that operator's system (the operator itself, its ``matvec``, the system ``SparseSym``, or
``None``), the whole iteration runs on the GPU (``bddc_pcg``: fused SpMV·dot, fused
axpy·norm, one host sync per iteration). Otherwise the reference recurrence runs on the
host around the given callables (which may themselves be device-backed).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .bddc import BddcOperator, NotSpdOperatorError
from .linalg import SparseSym, tridiag_eig


@dataclass
class SolveReport:
    """krylov.py:16-28."""

    iterations: int
    residual_history: list
    converged: bool
    kappa_estimate: float
    ritz_extremes: tuple
    alphas: list = None
    betas: list = None

    @property
    def relative_residual(self) -> float:
        if self.residual_history[0] == 0.0:
            return 0.0
        return self.residual_history[-1] / self.residual_history[0]


def _lanczos_extremes(alphas, betas):
    """Extreme Ritz values from the CG coefficients (krylov.py:95-104)."""
    k = len(alphas)
    diag = np.empty(k)
    off = np.empty(max(k - 1, 0))
    diag[0] = 1.0 / alphas[0]
    for j in range(1, k):
        diag[j] = 1.0 / alphas[j] + betas[j - 1] / alphas[j - 1]
        off[j - 1] = math.sqrt(betas[j - 1]) / alphas[j - 1]
    return tridiag_eig(diag, off)


def _report(alphas, betas, history, converged):
    if len(alphas) == 0:
        return SolveReport(0, list(history), converged, float("nan"), (float("nan"),) * 2, [], [])
    ritz = _lanczos_extremes(alphas, betas)
    kappa = ritz[1] / ritz[0] if ritz[0] > 0 else float("inf")
    return SolveReport(len(alphas), list(history), converged, kappa, ritz, list(alphas), list(betas))


def _device_operator(apply_A, apply_B):
    """The device operator if (apply_A, apply_B) is (its system, it); else None."""
    if isinstance(apply_B, BddcOperator):
        op = apply_B
    elif getattr(apply_B, "__func__", None) is BddcOperator.apply:
        op = apply_B.__self__
    else:
        return None
    if apply_A is None or apply_A is op or getattr(apply_A, "__self__", None) is op:
        return op
    if isinstance(apply_A, SparseSym) and apply_A is op.system._matrix:
        return op
    return None


def pcg(apply_A, apply_B, b, tol: float = 1e-6, max_iters: int = 2000):
    """Solve A x = b with preconditioner B from x0 = 0 (krylov.py:31-92)."""
    op = _device_operator(apply_A, apply_B)
    if op is not None:
        x, alphas, betas, hist, k, conv = op.pcg(b, tol=tol, max_iters=max_iters)
        if hist[0] == 0.0:
            return x, SolveReport(0, [0.0], True, float("nan"), (float("nan"),) * 2, [], [])
        return x, _report(list(alphas), list(betas), list(hist), conv)
    return _host_pcg(apply_A, apply_B, b, tol, max_iters)


def _host_pcg(apply_A, apply_B, b, tol, max_iters):
    if isinstance(apply_A, SparseSym):
        A = apply_A
        apply_A = A.matvec
    b = np.asarray(b, dtype=float)
    x = np.zeros_like(b)
    r = b.copy()
    norm0 = float(np.linalg.norm(r))
    history = [norm0]
    if norm0 == 0.0:
        return x, SolveReport(0, history, True, float("nan"), (float("nan"),) * 2, [], [])
    z = np.asarray(apply_B(r))
    rz = float(r @ z)
    if rz <= 0.0:
        raise NotSpdOperatorError(f"preconditioner not SPD: <r, Br> = {rz}")
    p = z.copy()
    alphas, betas = [], []
    converged = False
    for _ in range(max_iters):
        Ap = np.asarray(apply_A(p))
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            raise NotSpdOperatorError(f"operator not SPD: <p, Ap> = {pAp}")
        alpha = rz / pAp
        alphas.append(alpha)
        x += alpha * p
        r -= alpha * Ap
        rnorm = float(np.linalg.norm(r))
        history.append(rnorm)
        if rnorm <= tol * norm0:
            converged = True
            break
        z = np.asarray(apply_B(r))
        rz_new = float(r @ z)
        if rz_new <= 0.0:
            raise NotSpdOperatorError(f"preconditioner not SPD: <r, Br> = {rz_new}")
        beta = rz_new / rz
        betas.append(beta)
        rz = rz_new
        p = z + beta * p
    return x, _report(alphas, betas, history, converged)
