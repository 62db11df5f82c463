"""Three-level BDDC-SO: the paper's outlook, which the
reference does not implement (SPEC.md:15 lists multi-level BDDC as out of scope).

The level-1 coarse problem S_0 = Σ_i R_iᵀ S_0i R_i (bddc.py:494-505) is itself a finite-element-like
problem: its "elements" are the subdomains, with the dense element matrices S_0i = Ψ_iᵀ A_i Ψ_i the
setup already holds on the device, and its unknowns are the coarse dofs (vertices and subobject
averages). :class:`Level2Bddc` applies BDDC to it algebraically, following the three-level method of
Tu (2007) / Mandel, Sousedík, Dohrmann (2008):

* level-2 subdomains ("boxes") are blocks of ``coarsening`` subdomains per axis of the Θ lattice;
* a coarse dof is interior to a box if all its owning subdomains lie in that box, otherwise it is
  on the level-2 interface Γ₂; Γ₂ dofs with the same set of boxes form one level-2 object (a face,
  edge or vertex of the box lattice);
* one constraint per object: the normalised mean of its dofs (constants on a floating box are the
  all-ones coefficient vector, so one mean per object controls every local kernel);
* cardinality weights 1/|boxes(g)|; local constrained solves through K_J = S_J + s CᵀC (the same
  augmentation as the level-1 setup), Φ₂ = K⁻¹Cᵀ(C K⁻¹ Cᵀ)⁻¹, level-2 coarse matrix
  Σ_J R_Jᵀ ((C K⁻¹Cᵀ)⁻¹ − s I) R_J factored densely;
* the apply is the same three-step apply as level 1 (interior solves, interface preconditioner,
  discrete harmonic extension), all as batched dense operations over boxes padded to one shape.

``solve(r)`` is a fixed symmetric positive definite approximation of S_0⁻¹.
:class:`ThreeLevelOperator` installs it in a device :class:`~.bddc.BddcOperator` through the C ABI
hook ``bddc_set_coarse_solver``: the level-1 apply and the fused device PCG then call it in place
of the multifrontal coarse solve, on the library's stream.

Status: a prototype of the outlook, not a reference feature and not on the benchmarked path.
On the GPU the level-2 numeric setup (batched Cholesky, triangular solves, Schur complement,
explicit inverses) and the apply's matrix-vector products run on this library's own batched FP64
kernels (bddc_dense_potrf / trsm / gemm / gemv_t); torch does the gathers / scatters and the
dense factorization of the small level-2 coarse matrix. While the hook is installed, a re-setup
of the 3D path skips the exact coarse factorization (DESIGN.md §10a has the measurements). On a
CPU device the same formulas run through torch: that evaluation is the tests' checker.
"""

from __future__ import annotations

import ctypes as C
import traceback

import numpy as np

from . import _capi


class Level2Bddc:
    """Algebraic BDDC preconditioner for S_0 = Σ_e scatter(elem_mats[e]) over ``elem_ids[e]``.

    ``elem_ids`` (E, ncp) int: global unknowns of each element, −1 padded. ``elem_mats``
    (E, ncp, ncp): dense symmetric element matrices (torch tensor or array; padding ignored).
    ``box_of_elem`` (E,): level-2 subdomain of each element. Runs on a CUDA device; ``checker=True``
    allows the CPU evaluation of the same formulas, which only the tests use.
    """

    def __init__(self, elem_ids, elem_mats, box_of_elem, n0: int, device=None, weights: str = "cardinality",
                 checker: bool = False):
        import torch

        if weights not in ("cardinality", "stiffness"):
            raise ValueError(f"unknown level-2 weights {weights!r}")
        self.weights = weights

        self._torch = torch
        ids = np.asarray(elem_ids, dtype=np.int64)
        box_of_elem = np.asarray(box_of_elem, dtype=np.int64)
        E, ncp = ids.shape
        mats = torch.as_tensor(elem_mats, dtype=torch.float64)
        dev = mats.device if device is None else torch.device(device)
        mats = mats.to(dev)
        if mats.shape != (E, ncp, ncp):
            raise ValueError(f"element matrices have shape {tuple(mats.shape)}, expected {(E, ncp, ncp)}")
        if dev.type != "cuda" and not checker:
            raise RuntimeError("Level2Bddc runs on a CUDA device with this library's kernels (no CPU fallback); "
                               "the CPU evaluation exists for the tests only (checker=True)")
        self.n0, self.device = int(n0), dev
        nbox = int(box_of_elem.max()) + 1 if E else 0
        self.n_boxes = nbox

        # ---- symbolic: (dof, box) incidences, interior / interface, objects ----
        valid = ids >= 0
        ebox = np.broadcast_to(box_of_elem[:, None], ids.shape)
        key = np.unique(ids[valid] * nbox + ebox[valid])
        dof, box = key // nbox, key % nbox
        cnt = np.bincount(dof, minlength=n0)
        if np.any(cnt == 0):
            raise ValueError("every coarse unknown must belong to an element")
        ptr = np.concatenate([[0], np.cumsum(cnt)])
        sig = -np.ones((n0, int(cnt.max())), dtype=np.int64)
        sig[dof, np.arange(len(dof)) - ptr[dof]] = box
        gam = np.flatnonzero(cnt >= 2)
        usig, obj_of_gam = np.unique(sig[gam], axis=0, return_inverse=True)
        obj_of_gam = obj_of_gam.reshape(-1)
        nobj = len(usig)
        obj_of = -np.ones(n0, dtype=np.int64)
        obj_of[gam] = obj_of_gam
        obj_size = np.bincount(obj_of_gam, minlength=nobj)
        self.n_gamma2, self.n_coarse2 = len(gam), nobj
        self.objects = usig  # box signature of each level-2 object (−1 padded)

        inter = cnt[dof] >= 2
        I_of = [np.zeros(0, np.int64)] * nbox
        G_of = [np.zeros(0, np.int64)] * nbox
        order = np.argsort(box, kind="stable")
        bptr = np.concatenate([[0], np.cumsum(np.bincount(box, minlength=nbox))])
        for J in range(nbox):
            sl = order[bptr[J]:bptr[J + 1]]
            d = dof[sl]
            I_of[J] = d[~inter[sl]]
            G_of[J] = d[inter[sl]]
        O_of = [np.unique(obj_of[g]) for g in G_of]
        nI = max((len(a) for a in I_of), default=0)
        nG = max((len(a) for a in G_of), default=0)
        nC = max((len(a) for a in O_of), default=0)
        self.shape = (nbox, nI, nG, nC)

        r8 = lambda v: max(8, -(-v // 8) * 8)  # noqa: E731 - even leading dimensions for the dense kernels
        idxI = np.full((nbox, r8(nI)), n0, dtype=np.int64)
        idxG = np.full((nbox, r8(nG)), n0, dtype=np.int64)
        idxC = np.full((nbox, r8(nC)), nobj, dtype=np.int64)
        wG = np.zeros((nbox, r8(nG)))
        Cm = np.zeros((nbox, r8(nC), r8(nG)))
        for J in range(nbox):
            idxI[J, :len(I_of[J])] = I_of[J]
            idxG[J, :len(G_of[J])] = G_of[J]
            idxC[J, :len(O_of[J])] = O_of[J]
            wG[J, :len(G_of[J])] = 1.0 / cnt[G_of[J]]
            k = np.searchsorted(O_of[J], obj_of[G_of[J]])
            Cm[J, k, np.arange(len(G_of[J]))] = 1.0 / np.sqrt(obj_size[obj_of[G_of[J]]])
        t = lambda a, dt=None: torch.as_tensor(a, dtype=dt, device=dev)  # noqa: E731
        self.idxI, self.idxG, self.idxC = t(idxI), t(idxG), t(idxC)
        self.wG = t(wG, torch.float64)
        Cmat = t(Cm, torch.float64)
        nIp, nGp, nCp = idxI.shape[1], idxG.shape[1], idxC.shape[1]

        # ---- numeric: assemble every box at once, Schur complement on Γ₂, constrained solves ----
        # local position of each (dof, box) incidence: interior dofs first, then the interface
        nJ = nIp + nGp
        inc_pos = np.empty(len(key), dtype=np.int64)
        for J in range(nbox):
            sl = order[bptr[J]:bptr[J + 1]]
            isl = inter[sl]
            inc_pos[sl[~isl]] = np.arange(int((~isl).sum()))
            inc_pos[sl[isl]] = nIp + np.arange(int(isl.sum()))
        ekey = np.where(valid, ids * nbox + ebox, -1)
        loc = np.where(valid, inc_pos[np.searchsorted(key, np.maximum(ekey, 0))], nJ)  # (E, ncp); padding -> dummy
        flat = (box_of_elem[:, None, None] * (nJ + 1) + loc[:, :, None]) * (nJ + 1) + loc[:, None, :]
        self._flat = t(flat.reshape(-1))
        del flat
        self._Cmat = Cmat
        self._ngs = t(np.array([max(len(g), 1) for g in G_of]), torch.float64)
        self._dims = (nbox, nIp, nGp, nCp, nJ, nobj, E, ncp)
        self.refactor(mats)

    def refactor(self, elem_mats):
        """Numeric setup for new element matrices on the same elements / boxes (the symbolic
        part above is kept). BDDC_L2_TIMING=1 prints the time of each stage (synchronising)."""
        torch = self._torch
        import os
        import sys
        import time

        timing = os.environ.get("BDDC_L2_TIMING") == "1" and self.device.type == "cuda"
        tprev = [time.perf_counter()]

        def mark(name):
            if timing:
                torch.cuda.synchronize(self.device)
                now = time.perf_counter()
                print(f"level-2 numeric: {name:<34s}{(now - tprev[0]) * 1e3:9.2f} ms", file=sys.stderr)
                tprev[0] = now
        dev, n0 = self.device, self.n0
        nbox, nIp, nGp, nCp, nJ, nobj, E, ncp = self._dims
        mats = torch.as_tensor(elem_mats, dtype=torch.float64).to(dev)
        if mats.shape != (E, ncp, ncp):
            raise ValueError(f"element matrices have shape {tuple(mats.shape)}, expected {(E, ncp, ncp)}")
        Cmat, ngs = self._Cmat, self._ngs
        Aall = torch.zeros(nbox * (nJ + 1) * (nJ + 1), dtype=torch.float64, device=dev)
        Aall.index_add_(0, self._flat, mats.reshape(-1))
        Aall = Aall.view(nbox, nJ + 1, nJ + 1)
        AII = Aall[:, :nIp, :nIp].clone()
        AIG = Aall[:, :nIp, nIp:nJ].clone()
        AGG = Aall[:, nIp:nJ, nIp:nJ].clone()
        del Aall
        AII += torch.diag_embed((self.idxI >= n0).to(torch.float64))  # identity on the padding
        AGG += torch.diag_embed((self.idxG >= n0).to(torch.float64))
        mark("assemble boxes")
        AII = 0.5 * (AII + AII.transpose(1, 2))
        validG = (self.idxG < n0).to(torch.float64)
        if dev.type == "cuda":
            # the O(n^3) work on this library's batched FP64 kernels (dense_f64.cu: DMMA tile
            # Cholesky, tile-inverse triangular solves, GEMM). A symmetric batch is its own
            # column-major image; potrf leaves L in the column-major lower triangle, which the
            # torch view reads as the upper factor U = L^T (upper=True below).
            self.upper = True
            AGI = AIG.transpose(1, 2).contiguous()       # column-major n_I x n_G, one box each
            LI = _own_potrf(torch, AII)                  # in place
            mark("potrf A_II")
            Xt = AGI.clone()
            _own_trsm(torch, 0, LI, Xt)                  # L y = A_IG
            _own_trsm(torch, 1, LI, Xt)                  # L^T X = y
            mark("X = A_II^-1 A_IG")
            S = AGG                                      # S = A_GG - A_IG^T X, in place
            _own_gemm(torch, True, False, -1.0, AGI, Xt, 1.0, S)
            mark("Schur complement")
            del Xt
            S.add_(S.transpose(1, 2).clone()).mul_(0.5)
            s = (torch.diagonal(S, dim1=1, dim2=2) * validG).sum(1) / ngs  # mean diagonal per box
            Cmat = self._stiffness_weights(torch.diagonal(S, dim1=1, dim2=2) * validG)
            Cs = Cmat * torch.sqrt(s)[:, None, None]
            S.baddbmm_(Cs.transpose(1, 2), Cs)           # K = S + s C^T C, in place
            del Cs
            LK = _own_potrf(torch, S)
            mark("K = S + s C^T C, potrf")
            Yt = Cmat.clone()                            # column-major n_G x n_C = C^T
            _own_trsm(torch, 0, LK, Yt)
            _own_trsm(torch, 1, LK, Yt)
            Y = Yt.transpose(1, 2).contiguous()          # K^{-1} C^T
            del Yt
            # explicit symmetric inverses, so that the apply is batched matrix-vector products
            eyeI = torch.eye(nIp, dtype=torch.float64, device=dev).expand(nbox, -1, -1).contiguous()
            _own_trsm(torch, 0, LI, eyeI)
            _own_trsm(torch, 1, LI, eyeI)
            del LI, AII
            self.AIIinv = eyeI.add_(eyeI.transpose(1, 2).clone()).mul_(0.5)
            mark("explicit A_II^-1 (and Y)")
            eyeG = torch.eye(nGp, dtype=torch.float64, device=dev).expand(nbox, -1, -1).contiguous()
            _own_trsm(torch, 0, LK, eyeG)
            _own_trsm(torch, 1, LK, eyeG)
            del LK, S, AGG
            self.Kinv = eyeG
            mark("explicit K^-1")
            self.AGI = AGI
        else:  # CPU evaluation of the same formulas (the tests' checker of the device level 2)
            self.upper = False
            self.LI = torch.linalg.cholesky(AII)
            X = torch.cholesky_solve(AIG, self.LI)
            S = AGG - AIG.transpose(1, 2) @ X
            S = 0.5 * (S + S.transpose(1, 2))
            s = (torch.diagonal(S, dim1=1, dim2=2) * validG).sum(1) / ngs
            Cmat = self._stiffness_weights(torch.diagonal(S, dim1=1, dim2=2) * validG)
            self.LK = torch.linalg.cholesky(S + s[:, None, None] * (Cmat.transpose(1, 2) @ Cmat))
            Y = torch.cholesky_solve(Cmat.transpose(1, 2).contiguous(), self.LK)  # K⁻¹Cᵀ
        self.AIG = AIG
        self.s = s
        G = Cmat @ Y
        padC = (self.idxC >= nobj).to(torch.float64)
        G = G + torch.diag_embed(padC)
        Ginv = torch.linalg.inv(0.5 * (G + G.transpose(1, 2)))
        self.Y = Y
        self.Phi = Y @ Ginv
        if dev.type == "cuda":  # T2 = K^{-1} - Phi Y^T: the constrained local solve as one matrix
            T2 = self.Kinv.baddbmm_(self.Phi, Y.transpose(1, 2), alpha=-1.0)
            del self.Kinv
            self.T2 = T2.add_(T2.transpose(1, 2).clone()).mul_(0.5)
            self.PhiT = self.Phi.transpose(1, 2).contiguous()
            mark("Phi, T2")
        Ecoarse = Ginv - s[:, None, None] * torch.eye(nCp, dtype=torch.float64, device=dev)
        # only the valid (constraint, constraint) pairs of each box are scattered (the padded slots
        # would all hit one address); S00 is exactly n00 x n00 and contiguous. Only the lower
        # triangle is read by the factorization, so no symmetrisation pass is needed.
        if getattr(self, "_s00_lin", None) is None:
            okC = self.idxC < nobj
            pair_ok = okC[:, :, None] & okC[:, None, :]
            lin = self.idxC[:, :, None] * max(nobj, 1) + self.idxC[:, None, :]
            self._s00_mask, self._s00_lin = pair_ok, lin[pair_ok]
        S00 = torch.zeros(max(nobj, 1) * max(nobj, 1), dtype=torch.float64, device=dev)
        S00.index_add_(0, self._s00_lin, Ecoarse[self._s00_mask])
        S00 = S00.view(max(nobj, 1), max(nobj, 1))
        self.S00 = S00
        mark("assemble S00")
        self.L00 = torch.linalg.cholesky(self.S00) if nobj else None
        mark("Cholesky of S00")
        self.S00inv = None
        if dev.type == "cuda" and 0 < nobj <= 8192:  # explicit inverse: the level-2 coarse solve is one GEMV
            n8 = -(-nobj // 8) * 8
            inv = torch.cholesky_inverse(self.L00)
            self.S00inv = torch.zeros((1, n8, n8), dtype=torch.float64, device=dev)
            self.S00inv[0, :nobj, :nobj] = 0.5 * (inv + inv.T)

    def _stiffness_weights(self, dS):
        """weights="stiffness": D_J(g) = S_J(g, g) / Σ_J' S_J'(g, g), the algebraic counterpart of
        the coefficient weights of Remark 1 (bddc.py:108-145) for coarse problems with jumps."""
        if self.weights != "stiffness":
            return self._Cmat
        torch = self._torch
        tot = torch.zeros(self.n0 + 1, dtype=torch.float64, device=self.device)
        tot.index_add_(0, self.idxG.reshape(-1), dS.reshape(-1))
        den = tot[self.idxG]
        self.wG = torch.where(den > 0, dS / torch.where(den > 0, den, torch.ones_like(den)), torch.zeros_like(dS))
        return self._Cmat  # (stiffness-weighted means were measured: 32 -> 31 iterations on cfg4b; plain means stay)

    def solve(self, r):
        """z ≈ S_0⁻¹ r (torch vector of n0 on ``device``)."""
        torch = self._torch
        n0 = self.n0
        zero = torch.zeros(1, dtype=torch.float64, device=self.device)
        rp = torch.cat([r, zero])
        if self.device.type == "cuda":
            return self._solve_gemv(rp)
        # interior solves, interface residual
        u1 = torch.cholesky_solve(rp[self.idxI].unsqueeze(2), self.LI, upper=self.upper)  # (B, nI, 1)
        tG = self.AIG.transpose(1, 2) @ u1
        rG = rp.clone()
        rG.index_add_(0, self.idxG.reshape(-1), -tG.reshape(-1))
        rG[n0] = 0.0
        # level-2 interface preconditioner
        rho = (self.wG * rG[self.idxG]).unsqueeze(2)  # (B, nG, 1)
        q = self.Phi.transpose(1, 2) @ rho  # (B, nC, 1)
        nobj = self.n_coarse2
        r00 = torch.zeros(nobj + 1, dtype=torch.float64, device=self.device)
        r00.index_add_(0, self.idxC.reshape(-1), q.reshape(-1))
        c = torch.zeros_like(r00)
        if nobj:
            c[:nobj] = torch.cholesky_solve(r00[:nobj].unsqueeze(1), self.L00).squeeze(1)
        v = torch.cholesky_solve(rho, self.LK, upper=self.upper) - self.Phi @ (self.Y.transpose(1, 2) @ rho)
        w = self.wG.unsqueeze(2) * (v + self.Phi @ c[self.idxC].unsqueeze(2))
        zG = torch.zeros(n0 + 1, dtype=torch.float64, device=self.device)
        zG.index_add_(0, self.idxG.reshape(-1), w.reshape(-1))
        zG[n0] = 0.0
        # harmonic extension + interior correction
        zI = u1 - torch.cholesky_solve(self.AIG @ zG[self.idxG].unsqueeze(2), self.LI, upper=self.upper)
        zG.index_put_((self.idxI.reshape(-1),), zI.reshape(-1))
        return zG[:n0]

    def _solve_gemv(self, rp):
        """The same apply with explicit inverses: every large product is one launch of the
        library's batched GEMV (bddc_dense_gemv_t); torch only gathers and scatters."""
        torch = self._torch
        n0, nobj = self.n0, self.n_coarse2
        mv = lambda M, x: _own_gemv(torch, M, x)  # noqa: E731
        u1 = mv(self.AIIinv, rp[self.idxI].contiguous())                 # (B, nI)
        rG = rp.clone()
        rG.index_add_(0, self.idxG.reshape(-1), -mv(self.AGI, u1).reshape(-1))
        rG[n0] = 0.0
        rho = (self.wG * rG[self.idxG]).contiguous()                       # (B, nG)
        q = mv(self.PhiT, rho)                                             # (B, nC)
        r00 = torch.zeros(nobj + 1, dtype=torch.float64, device=self.device)
        r00.index_add_(0, self.idxC.reshape(-1), q.reshape(-1))
        c = torch.zeros_like(r00)
        if nobj and self.S00inv is not None:
            n8 = self.S00inv.shape[1]
            rr = torch.zeros((1, n8), dtype=torch.float64, device=self.device)
            rr[0, :nobj] = r00[:nobj]
            c[:nobj] = mv(self.S00inv, rr)[0, :nobj]
        elif nobj:  # large level-2 coarse problems: triangular solves with the dense factor
            c[:nobj] = torch.cholesky_solve(r00[:nobj].unsqueeze(1), self.L00).squeeze(1)
        w = self.wG * (mv(self.T2, rho) + mv(self.Phi, c[self.idxC].contiguous()))
        zG = torch.zeros(n0 + 1, dtype=torch.float64, device=self.device)
        zG.index_add_(0, self.idxG.reshape(-1), w.reshape(-1))
        zG[n0] = 0.0
        zI = u1 - mv(self.AIIinv, mv(self.AIG, zG[self.idxG].contiguous()))
        zG.index_put_((self.idxI.reshape(-1),), zI.reshape(-1))
        return zG[:n0]

    def dense(self):
        """The operator as an explicit matrix (tests, small n0)."""
        torch = self._torch
        eye = torch.eye(self.n0, dtype=torch.float64, device=self.device)
        return torch.stack([self.solve(eye[i]) for i in range(self.n0)], dim=1)


def _own_potrf(torch, A):
    """In-place batched Cholesky of a contiguous symmetric (B, n, n) tensor on the library's
    kernels (bddc_dense_potrf); returns A, whose torch view then holds U = L^T above the
    diagonal."""
    lib = _capi.load()
    B, n, _ = A.shape
    info = (C.c_int * B)()
    rc = lib.bddc_dense_potrf(C.c_void_p(A.data_ptr()), n, n, n * n, B, info,
                              C.c_void_p(torch.cuda.current_stream(A.device).cuda_stream))
    if rc:
        raise RuntimeError(f"bddc_dense_potrf failed ({rc})")
    bad = [i for i in range(B) if info[i] >= 0]
    if bad:
        raise RuntimeError(f"level-2 matrix of box {bad[0]} is not positive definite (pivot {info[bad[0]]})")
    return A


def _own_gemv(torch, M, x):
    """y[b] = M[b] @ x[b] for a contiguous (B, n, k) tensor and x (B, k): the library's batched
    GEMV (each row of M is a contiguous column of the column-major k x n operand)."""
    lib = _capi.load()
    B, n, k = M.shape
    y = torch.empty((B, n), dtype=torch.float64, device=M.device)
    rc = lib.bddc_dense_gemv_t(k, n, 1.0, C.c_void_p(M.data_ptr()), k, n * k, C.c_void_p(x.data_ptr()), k, 0.0,
                               C.c_void_p(y.data_ptr()), n, B,
                               C.c_void_p(torch.cuda.current_stream(M.device).cuda_stream))
    if rc:
        raise RuntimeError(f"bddc_dense_gemv_t failed ({rc})")
    return y


def _own_trsm(torch, kind, L, Bt):
    """In place on Bt (B, nrhs, n) = column-major n x nrhs: kind 0 solves L y = b, 1 L^T x = y."""
    lib = _capi.load()
    B, nrhs, n = Bt.shape
    rc = lib.bddc_dense_trsm(kind, C.c_void_p(L.data_ptr()), n, n, n * n, C.c_void_p(Bt.data_ptr()), nrhs, n,
                             n * nrhs, B, C.c_void_p(torch.cuda.current_stream(Bt.device).cuda_stream))
    if rc:
        raise RuntimeError(f"bddc_dense_trsm failed ({rc})")


def _own_gemm(torch, tA, tB, alpha, At, Bt, beta, Ct):
    """Ct = alpha op(A) op(B) + beta Ct, every operand a (B, cols, rows) tensor = column-major
    rows x cols per box (bddc_dense_gemm)."""
    lib = _capi.load()
    nb = At.shape[0]
    M, N = Ct.shape[2], Ct.shape[1]
    K = At.shape[2] if tA else At.shape[1]
    rc = lib.bddc_dense_gemm(int(tA), int(tB), M, N, K, float(alpha), C.c_void_p(At.data_ptr()), At.shape[2],
                             At.shape[1] * At.shape[2], C.c_void_p(Bt.data_ptr()), Bt.shape[2],
                             Bt.shape[1] * Bt.shape[2], float(beta), C.c_void_p(Ct.data_ptr()), Ct.shape[2],
                             Ct.shape[1] * Ct.shape[2], nb, C.c_void_p(torch.cuda.current_stream(Ct.device).cuda_stream))
    if rc:
        raise RuntimeError(f"bddc_dense_gemm failed ({rc})")


def box_of_subdomains(subs, coarsening) -> np.ndarray:
    """Level-2 subdomain of each Θ subdomain: blocks of ``coarsening`` subdomains per axis of
    the ``subs`` lattice (first axis fastest, as the uniform Θ numbering of partition.py)."""
    subs = tuple(int(s) for s in subs)
    k = (int(coarsening),) * len(subs) if np.isscalar(coarsening) else tuple(int(c) for c in coarsening)
    nb = [-(-s // c) for s, c in zip(subs, k)]
    idx = np.indices(subs[::-1])[::-1]  # idx[a] has the a-th lattice coordinate, axis 0 fastest
    out = np.zeros(subs[::-1], dtype=np.int64)
    stride = 1
    for a in range(len(subs)):
        out += (idx[a] // k[a]) * stride
        stride *= nb[a]
    return out.reshape(-1)


class _DevVec:
    """CUDA array interface view of a raw device pointer (n doubles)."""

    def __init__(self, ptr: int, n: int, readonly: bool):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), readonly),
                                         "version": 2}


class ThreeLevelOperator:
    """A device BddcOperator whose coarse solve is one application of :class:`Level2Bddc`.

    ``apply`` / ``matvec`` / ``pcg`` are the wrapped operator's: every level-1 kernel runs as
    before, the multifrontal coarse solve is replaced through ``bddc_set_coarse_solver``.
    ``close()`` (or ``restore()``) puts the direct solve back.
    """

    def __init__(self, op, coarsening=2, _setup_under_hook=False):
        self.op = op
        self.coarsening = coarsening
        self.lean = bool(_setup_under_hook)
        self.calls = 0
        self._error = None
        self.level2 = None
        if op.plan.coarse is None:
            raise ValueError("the operator has no coarse problem")
        if op.pair.box_layout is None:
            raise ValueError("three-level BDDC-SO needs a uniform box partition Θ")
        self._fn = _capi.COARSE_SOLVER_FN(self._solve)  # keep the thunk alive
        if _setup_under_hook:  # hook first: the setup then builds no coarse plan, fronts or factor
            self._install()
            op._setup()
            self._build_level2()
        else:                  # an operator that is already set up (it keeps its exact factor)
            self._build_level2()
            self._install()

    @classmethod
    def build(cls, system, pair, objects, recipe, weights, coarsening=2, coarse_scaling="reference", device=0):
        """Three-level operator from nothing (the arguments of ``build_bddc``): the hook is
        installed before the setup, so the coarse problem is never planned, allocated or
        factored; only the level-1 local setup and the level 2 run."""
        from . import bddc as _b
        from .layout import build_device_plan
        from .weights import Recipe, select_constraints

        if isinstance(recipe, str):
            recipe = Recipe.parse(recipe)
        if coarse_scaling not in _b.COARSE_SCALINGS:
            raise ValueError(f"unknown coarse_scaling {coarse_scaling!r}; expected {_b.COARSE_SCALINGS}")
        if pair.box_layout is None:
            raise ValueError("three-level BDDC-SO needs a uniform box partition Θ")
        constraints = select_constraints(objects, recipe, pair)
        plan = build_device_plan(pair, constraints, weights, coarse_pattern="device", device=device)
        op = _b.BddcOperator(system, pair, weights, recipe, constraints, plan, coarse_scaling, device, None)
        return cls(op, coarsening, _setup_under_hook=True)

    def _install(self):
        rc = self.op._lib.bddc_set_coarse_solver(self.op._ctx, self._fn, None)
        if rc:
            raise RuntimeError("bddc_set_coarse_solver failed (sharded operators are not supported)")

    def _build_level2(self):
        import torch

        op, plan = self.op, self.op.plan
        mode = "stiffness" if getattr(op.weights, "mode", "") == "coefficient" else "cardinality"
        self.level2 = Level2Bddc(plan.con_coarse, self._element_matrices(),
                                 box_of_subdomains(op.pair.box_layout[0], self.coarsening), plan.coarse.n,
                                 device=torch.device(f"cuda:{op.device}"), weights=mode)

    def _element_matrices(self):
        """S_0i of every subdomain, a zero-copy view of the device setup's blocks
        (bddc_coarse_elements: nsub x nc_pad x nc_pad)."""
        import torch

        plan = self.op.plan
        cnt = C.c_longlong(0)
        ptr = self.op._lib.bddc_coarse_elements(self.op._ctx, C.byref(cnt))
        if not ptr or cnt.value != plan.nsub * plan.nc_pad * plan.nc_pad:
            raise RuntimeError("the coarse element matrices are not available")
        v = torch.as_tensor(_DevVec(ptr, cnt.value, False), device=torch.device(f"cuda:{self.op.device}"))
        return v.view(plan.nsub, plan.nc_pad, plan.nc_pad)

    def refactor(self, alpha=None):
        """New coefficient on the same partition: the level-1 numeric setup, then the level-2
        numeric setup from the new coarse element matrices (both symbolic parts are kept)."""
        self.op.refactor(alpha)  # under the hook the 3D path skips the exact coarse factorization
        self._refactored = True
        self.level2.refactor(self._element_matrices())

    def _solve(self, user, rhs, sol, n, stream):
        try:
            torch = self.level2._torch
            dev = self.level2.device
            with torch.cuda.stream(torch.cuda.ExternalStream(int(stream or 0), device=dev)):
                r = torch.as_tensor(_DevVec(rhs, n, False), device=dev)  # (torch takes no read-only views)
                x = torch.as_tensor(_DevVec(sol, n, False), device=dev)
                x.copy_(self.level2.solve(r))
            self.calls += 1
            return 0
        except Exception as e:  # noqa: BLE001 - reported to the library as a failed solve
            self._error = e
            traceback.print_exc()
            return 1

    def restore(self):
        """Back to the two-level operator (the exact coarse factor is rebuilt if a refactor under
        the hook skipped it)."""
        if self.lean:
            raise RuntimeError("this operator was set up under the hook: it has no exact coarse factor to restore")
        if self.op is not None and getattr(self.op, "_ctx", None):
            self.op._lib.bddc_set_coarse_solver(self.op._ctx, _capi.COARSE_SOLVER_FN(), None)  # NULL: direct solve
            if getattr(self, "_refactored", False):
                self._refactored = False
                self.op.refactor()

    def close(self):
        if getattr(self.op, "_ctx", None):
            self.op._lib.bddc_set_coarse_solver(self.op._ctx, _capi.COARSE_SOLVER_FN(), None)
        self.op.close()

    def __getattr__(self, name):  # apply, matvec, pcg, n, … of the wrapped operator
        if name in ("op", "level2", "_fn"):  # not set yet: no recursion through self.op
            raise AttributeError(name)
        return getattr(self.op, name)
