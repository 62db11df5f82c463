"""TEST INFRASTRUCTURE ONLY — numpy emulation of the sharded (multi-GPU) apply of
csrc/apply.cu + csrc/multigpu.cu, one process per rank over torch.distributed (gloo).

Every array a rank does not compute itself starts as NaN (poison). The only data moved
between ranks are the library's exchanges: the dof rows next to the cut lines (u1), every
rank's local coarse right-hand sides (allgather), and the interface values w of the
neighbours' boundary subdomain rows. A missing exchange therefore surfaces as NaN in the
result instead of a silently wrong number. Never imported by the product.
"""

from __future__ import annotations

import numpy as np


class GlooExchange:
    """The library's exchange set over torch.distributed (CPU tensors)."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world

    def _pair(self, send: np.ndarray, recv: np.ndarray, peer: int):
        import torch
        import torch.distributed as dist

        ts = torch.from_numpy(np.ascontiguousarray(send).ravel().copy())
        tr = torch.empty(recv.size, dtype=torch.float64)
        reqs = [dist.isend(ts, peer), dist.irecv(tr, peer)]
        for q in reqs:
            q.wait()
        recv[...] = tr.numpy().reshape(recv.shape)

    def dof_halo(self, v: np.ndarray, sl):
        if sl.lo_send >= 0:
            self._pair(v[sl.lo_send:sl.lo_send + sl.row_len], v[sl.lo_recv:sl.lo_recv + sl.row_len], self.rank - 1)
        if sl.hi_send >= 0:
            self._pair(v[sl.hi_send:sl.hi_send + sl.row_len], v[sl.hi_recv:sl.hi_recv + sl.row_len], self.rank + 1)

    def boundary_rows(self, per_sub: np.ndarray, sl):
        k = sl.sub_row
        if sl.lo_send >= 0:
            self._pair(per_sub[sl.s_lo:sl.s_lo + k], per_sub[sl.s_lo - k:sl.s_lo], self.rank - 1)
        if sl.hi_send >= 0:
            self._pair(per_sub[sl.s_hi - k:sl.s_hi], per_sub[sl.s_hi:sl.s_hi + k], self.rank + 1)

    def allgather_subs(self, per_sub: np.ndarray, slabs):
        import torch
        import torch.distributed as dist

        for r, s in enumerate(slabs):
            blk = per_sub[s.s_lo:s.s_hi]
            t = torch.from_numpy(np.ascontiguousarray(blk).copy())
            dist.broadcast(t, src=r)
            per_sub[s.s_lo:s.s_hi] = t.numpy().reshape(blk.shape)


def sharded_apply(em, plan, r_full: np.ndarray, sl, slabs, ex: GlooExchange) -> np.ndarray:
    """z = B r on this rank's slab (valid on its active rows), mirroring apply_bddc."""
    n = em.n
    A = em.A.copy()
    A.eliminate_zeros()  # explicit zeros would multiply poison
    nsub = plan.nsub
    gam = np.asarray(plan.gamma_dof, dtype=np.int64)
    gact = gam[(gam >= sl.f_lo) & (gam < sl.f_hi)]
    own = range(sl.s_lo, sl.s_hi)
    r = np.full(n, np.nan)
    r[sl.f_lo:sl.f_hi] = r_full[sl.f_lo:sl.f_hi]
    # u1 = A_II^{-1} r_I on own subdomains (zero on Gamma), then the cut-row halo
    u1 = np.full(n, np.nan)
    u1[gam] = 0.0
    for p in own:
        L = em.loc[p]
        fI = L["fid"][L["I"]]
        if len(fI):
            u1[fI] = np.linalg.solve(L["AII"], r[fI])
    ex.dof_halo(u1, sl)
    rp = np.full(n, np.nan)
    rp[gact] = r[gact] - A[gact] @ u1
    # local Gamma phase 1 on own subdomains; the coarse rhs blocks are allgathered
    ncmax = max(len(L["cc"]) for L in em.loc) if em.loc else 0
    qloc = np.full((nsub, max(ncmax, 1)), np.nan)
    st = {}
    for p in own:
        L = em.loc[p]
        g = L["gam"]
        rho = np.where(g >= 0, L["w"] * np.where(g >= 0, rp[L["fid"][L["Gn"]]], 0.0), 0.0)
        u = np.linalg.solve(L["LS"].T, np.linalg.solve(L["LS"], rho))
        t = L["C"] @ u
        q = L["c"] * (L["Phi"].T @ rho)
        qloc[p, :len(q)] = q
        st[p] = (u, t)
    ex.allgather_subs(qloc, slabs)
    ncoarse = em.cp.n if em.cp is not None else 0
    crhs = np.zeros(ncoarse)
    for p in range(nsub):  # subdomain order = the single-rank summation order
        cc = em.loc[p]["cc"]
        np.add.at(crhs, cc, qloc[p, :len(cc)])
    csol = em.coarse_solve(crhs) if ncoarse else crhs
    # local Gamma phase 2, neighbours' boundary rows, interface gather on the active rows
    nGmax = max(len(L["Gn"]) for L in em.loc)
    wloc = np.full((nsub, nGmax), np.nan)
    for p in own:
        L = em.loc[p]
        u, t = st[p]
        e = L["c"] * csol[L["cc"]] - t
        wloc[p, :len(u)] = L["w"] * (u + L["Phi"] @ e)
    ex.boundary_rows(wloc, sl)
    z = np.full(n, np.nan)
    z[gact] = 0.0
    lo, hi = sl.f_lo, sl.f_hi
    for p in range(nsub):
        L = em.loc[p]
        f = L["fid"][L["Gn"]]
        m = (f >= lo) & (f < hi)
        if m.any():
            np.add.at(z, f[m], wloc[p, :len(f)][m])
    # z_I = A_II^{-1} (r - A z_Gamma)_I on own subdomains (residuals before any solve)
    for p in own:
        L = em.loc[p]
        z[L["fid"][L["I"]]] = 0.0
    ys = {}
    for p in own:
        L = em.loc[p]
        fI = L["fid"][L["I"]]
        if len(fI):
            ys[p] = r[fI] - A[fI] @ z
    for p, y in ys.items():
        L = em.loc[p]
        z[L["fid"][L["I"]]] = np.linalg.solve(L["AII"], y)
    return z
