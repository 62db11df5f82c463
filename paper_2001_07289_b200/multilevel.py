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

Status: a prototype of the outlook, not a reference feature. On the GPU the level-2 setup's
factorizations, multi-right-hand-side triangular solves and Schur-complement product run on this
library's batched FP64 kernels (bddc_dense_potrf / trsm / gemm); the apply's single-vector solves
and the gathers / scatters go through torch (library kernels). It is not part of the benchmarked
path. On a CPU device the same formulas run through torch: that evaluation is the tests' checker. No reference exists to pin it: the tests check the
properties the method guarantees (symmetry, positive definiteness, a bounded condition number of
the preconditioned coarse problem, PCG convergence to the two-level solution).
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
    ``box_of_elem`` (E,): level-2 subdomain of each element. Works on any torch device in FP64.
    """

    def __init__(self, elem_ids, elem_mats, box_of_elem, n0: int, device=None):
        import torch

        self._torch = torch
        ids = np.asarray(elem_ids, dtype=np.int64)
        box_of_elem = np.asarray(box_of_elem, dtype=np.int64)
        E, ncp = ids.shape
        mats = torch.as_tensor(elem_mats, dtype=torch.float64)
        dev = mats.device if device is None else torch.device(device)
        mats = mats.to(dev)
        if mats.shape != (E, ncp, ncp):
            raise ValueError(f"element matrices have shape {tuple(mats.shape)}, expected {(E, ncp, ncp)}")
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

        # ---- numeric: assemble each box, Schur complement on Γ₂, constrained solves ----
        AII = torch.zeros((nbox, nIp, nIp), dtype=torch.float64, device=dev)
        AIG = torch.zeros((nbox, nIp, nGp), dtype=torch.float64, device=dev)
        AGG = torch.zeros((nbox, nGp, nGp), dtype=torch.float64, device=dev)
        eorder = np.argsort(box_of_elem, kind="stable")
        eptr = np.concatenate([[0], np.cumsum(np.bincount(box_of_elem, minlength=nbox))])
        pos = np.empty(n0 + 1, dtype=np.int64)
        for J in range(nbox):
            ni, ng = len(I_of[J]), len(G_of[J])
            nJ = nIp + nGp
            pos[:] = nJ  # dummy row / column for padding
            pos[I_of[J]] = np.arange(ni)
            pos[G_of[J]] = nIp + np.arange(ng)
            el = eorder[eptr[J]:eptr[J + 1]]
            loc = t(pos[np.where(ids[el] >= 0, ids[el], n0)])  # (m, ncp)
            A = torch.zeros((nJ + 1, nJ + 1), dtype=torch.float64, device=dev)
            A.index_put_((loc[:, :, None].expand(-1, -1, ncp), loc[:, None, :].expand(-1, ncp, -1)),
                         mats[t(el)], accumulate=True)
            AII[J], AIG[J], AGG[J] = A[:nIp, :nIp], A[:nIp, nIp:nJ], A[nIp:nJ, nIp:nJ]
            padI = torch.arange(ni, nIp, device=dev)
            AII[J, padI, padI] = 1.0
            padG = torch.arange(ng, nGp, device=dev)
            AGG[J, padG, padG] = 1.0
        AII = 0.5 * (AII + AII.transpose(1, 2))
        ngs = t(np.array([max(len(g), 1) for g in G_of]), torch.float64)
        validG = (self.idxG < n0).to(torch.float64)
        CtC = Cmat.transpose(1, 2) @ Cmat
        if dev.type == "cuda":
            # the O(n^3) work on this library's batched FP64 kernels (dense_f64.cu: DMMA tile
            # Cholesky, tile-inverse triangular solves, GEMM). A symmetric batch is its own
            # column-major image; potrf leaves L in the column-major lower triangle, which the
            # torch view reads as the upper factor U = L^T (upper=True below).
            self.upper = True
            self.LI = _own_potrf(torch, AII.contiguous())
            Xt = AIG.transpose(1, 2).contiguous()        # column-major n_I x n_G, one box each
            _own_trsm(torch, 0, self.LI, Xt)             # L y = A_IG
            _own_trsm(torch, 1, self.LI, Xt)             # L^T X = y
            S = AGG.contiguous()                         # S = A_GG - A_IG^T X
            _own_gemm(torch, True, False, -1.0, AIG.transpose(1, 2).contiguous(), Xt, 1.0, S)
            S = 0.5 * (S + S.transpose(1, 2))
            s = (torch.diagonal(S, dim1=1, dim2=2) * validG).sum(1) / ngs  # mean diagonal per box
            self.LK = _own_potrf(torch, (S + s[:, None, None] * CtC).contiguous())
            Yt = Cmat.clone()                            # column-major n_G x n_C = C^T
            _own_trsm(torch, 0, self.LK, Yt)
            _own_trsm(torch, 1, self.LK, Yt)
            Y = Yt.transpose(1, 2).contiguous()          # K^{-1} C^T
        else:  # CPU evaluation of the same formulas (the tests' checker of the device level 2)
            self.upper = False
            self.LI = torch.linalg.cholesky(AII)
            X = torch.cholesky_solve(AIG, self.LI)
            S = AGG - AIG.transpose(1, 2) @ X
            S = 0.5 * (S + S.transpose(1, 2))
            s = (torch.diagonal(S, dim1=1, dim2=2) * validG).sum(1) / ngs
            self.LK = torch.linalg.cholesky(S + s[:, None, None] * CtC)
            Y = torch.cholesky_solve(Cmat.transpose(1, 2).contiguous(), self.LK)  # K⁻¹Cᵀ
        self.AIG = AIG
        self.s = s
        G = Cmat @ Y
        padC = (self.idxC >= nobj).to(torch.float64)
        G = G + torch.diag_embed(padC)
        Ginv = torch.linalg.inv(0.5 * (G + G.transpose(1, 2)))
        self.Y = Y
        self.Phi = Y @ Ginv
        Ecoarse = Ginv - s[:, None, None] * torch.eye(nCp, dtype=torch.float64, device=dev)
        S00 = torch.zeros((nobj + 1, nobj + 1), dtype=torch.float64, device=dev)
        S00.index_put_((self.idxC[:, :, None].expand(-1, -1, nCp), self.idxC[:, None, :].expand(-1, nCp, -1)),
                       Ecoarse, accumulate=True)
        S00 = S00[:nobj, :nobj]
        self.S00 = 0.5 * (S00 + S00.T)
        self.L00 = torch.linalg.cholesky(self.S00) if nobj else None

    def solve(self, r):
        """z ≈ S_0⁻¹ r (torch vector of n0 on ``device``)."""
        torch = self._torch
        n0 = self.n0
        zero = torch.zeros(1, dtype=torch.float64, device=self.device)
        rp = torch.cat([r, zero])
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

    def __init__(self, op, coarsening=2):
        import torch

        self.op = op
        plan = op.plan
        if plan.coarse is None:
            raise ValueError("the operator has no coarse problem")
        if op.pair.box_layout is None:
            raise ValueError("three-level BDDC-SO needs a uniform box partition Θ")
        subs = op.pair.box_layout[0]
        nsub, ncp = plan.nsub, plan.nc_pad
        n0 = plan.coarse.n
        dev = torch.device(f"cuda:{op.device}")
        sloc = np.empty(nsub * ncp * ncp)
        got = op._lib.bddc_read_buffer(op._ctx, b"Sloc", 0, sloc.size, _capi.ptr(sloc, C.c_double))
        if got != sloc.size:
            raise RuntimeError("reading the coarse element matrices failed")
        self.level2 = Level2Bddc(plan.con_coarse, torch.from_numpy(sloc.reshape(nsub, ncp, ncp)),
                                 box_of_subdomains(subs, coarsening), n0, device=dev)
        self.calls = 0
        self._error = None
        self._fn = _capi.COARSE_SOLVER_FN(self._solve)  # keep the thunk alive
        rc = op._lib.bddc_set_coarse_solver(op._ctx, self._fn, None)
        if rc:
            raise RuntimeError("bddc_set_coarse_solver failed (sharded operators are not supported)")

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
        if self.op is not None and getattr(self.op, "_ctx", None):
            self.op._lib.bddc_set_coarse_solver(self.op._ctx, _capi.COARSE_SOLVER_FN(), None)  # NULL: direct solve

    def close(self):
        self.restore()
        self.op.close()

    def __getattr__(self, name):  # apply, matvec, pcg, n, … of the wrapped operator
        return getattr(self.op, name)
