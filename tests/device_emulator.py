"""TEST INFRASTRUCTURE ONLY — numpy emulation of the device algorithm over the same
host tables (DevicePlan), used to validate the index tables, the Schur / augmented
formulation and the multifrontal symbolic plan on CPU (no GPU in the build container).
Never imported by the product.
"""

from __future__ import annotations

import numpy as np

from paper_2001_07289_b200.mesh import assemble_cells


class Emulator:
    def __init__(self, system, pair, plan, coarse_scaling="reference"):
        mesh = system.mesh
        self.mesh, self.plan = mesh, plan
        lay = plan.layout
        subs, blk = pair.box_layout
        dim = mesh.dim
        nsub = plan.nsub
        self.A = system.matrix.tocsr()
        self.n = mesh.free_count
        self.loc = []
        Sblocks = []
        npd = np.asarray(blk) + 1
        nf = np.asarray(mesh.cells_per_dim) - 1
        for p in range(nsub):
            pc = [(p // int(np.prod(subs[:d]))) % subs[d] for d in range(dim)]
            # local nodes in layout order -> global free dofs
            ids = np.arange(lay.nloc_nodes)
            lc = np.zeros((lay.nloc_nodes, dim), dtype=np.int64)
            rem = ids.copy()
            for d in range(dim):
                lc[:, d] = rem % npd[d]
                rem //= npd[d]
            gc = lc + np.asarray(pc) * np.asarray(blk)
            dirich = np.any((gc == 0) | (gc == np.asarray(mesh.cells_per_dim)), axis=1)
            fid = np.zeros(lay.nloc_nodes, dtype=np.int64)
            st = 1
            for d in range(dim):
                fid += (gc[:, d] - 1) * st
                st *= int(nf[d])
            fid[dirich] = -1
            cells = np.flatnonzero(pair.theta == p)
            keep = np.flatnonzero(~dirich)
            Aloc = assemble_cells(mesh, system.coeff, cells, mesh.free_nodes[fid[keep]]).todense()
            full = np.zeros((lay.nloc_nodes, lay.nloc_nodes))
            full[np.ix_(keep, keep)] = Aloc
            s_i = float(np.mean(np.abs(np.diag(Aloc))))
            I_nodes = lay.irow_node[lay.irow_node >= 0]
            G_nodes = lay.slot_node
            AII = full[np.ix_(I_nodes, I_nodes)]
            AIG = full[np.ix_(I_nodes, G_nodes)]
            AGG = full[np.ix_(G_nodes, G_nodes)].copy()
            dG = dirich[G_nodes]
            AGG[dG, dG] = 1.0
            LI = np.linalg.cholesky(AII) if len(I_nodes) else np.zeros((0, 0))
            E = np.linalg.solve(LI, AIG) if len(I_nodes) else np.zeros((0, len(G_nodes)))
            SG = AGG - E.T @ E
            nG = lay.nG
            con = plan.slot_con[p, :nG]
            coef = plan.slot_coef[p, :nG]
            nc = int(plan.n_con_local[p])
            C = np.zeros((nc, nG))
            for s in range(nG):
                if con[s] >= 0:
                    C[con[s], s] = coef[s]
            SK = SG + s_i * C.T @ C
            LS = np.linalg.cholesky(SK)
            if nc:
                Gm = np.linalg.solve(LS, C.T)
                SC = Gm.T @ Gm
                Phi = np.linalg.solve(LS.T, Gm @ np.linalg.inv(SC))
                c = 1.0 / s_i**2 if coarse_scaling == "reference" else 1.0
                P = Phi.T @ SG @ Phi
                Sl = c * c * 0.5 * (P + P.T)
            else:
                Phi = np.zeros((nG, 0))
                c = 1.0
                Sl = np.zeros((0, 0))
            Sblocks.append(Sl)
            self.loc.append(dict(fid=fid, I=I_nodes, Gn=G_nodes, AII=AII, LS=LS, Phi=Phi, c=c,
                                 w=plan.slot_w[p, :nG], gam=plan.slot_gamma[p, :nG], C=C,
                                 cc=plan.con_coarse[p, :nc]))
        # coarse matrix in elimination order from local blocks (segmented sums)
        cp = plan.coarse
        self.cp = cp
        if cp is not None:
            ncp = plan.nc_pad
            flat = np.zeros(nsub * ncp * ncp)
            for p, Sl in enumerate(Sblocks):
                m = Sl.shape[0]
                blkp = np.zeros((ncp, ncp))
                blkp[:m, :m] = Sl
                flat[p * ncp * ncp:(p + 1) * ncp * ncp] = blkp.ravel(order="F")
            vals = np.add.reduceat(flat[cp.contrib], cp.seg_ptr[:-1]) if len(cp.contrib) else np.zeros(0)
            n = cp.n
            S0 = np.zeros((n, n))
            S0[cp.csr_row, cp.csr_col] = vals
            S0 = S0 + np.tril(S0, -1).T
            self.S0_elim = S0
            self._multifrontal(S0)

    def _multifrontal(self, S0):
        cp = self.cp
        N = cp.nnodes
        self.fronts = []
        upd = [None] * N
        for i in range(N):
            s0, s = cp.sep_start[i], cp.sep_size[i]
            bnd = cp.bnd_idx[cp.bnd_ptr[i]:cp.bnd_ptr[i + 1]]
            idx = np.concatenate([np.arange(s0, s0 + s), bnd])
            F = np.tril(S0[np.ix_(idx, idx)])
            F[s:, s:] = 0.0  # only the separator columns come from S_0 here
            for k in np.flatnonzero(cp.parent == i):
                rm = cp.rmap[cp.bnd_ptr[k]:cp.bnd_ptr[k + 1]]
                F[np.ix_(rm, rm)] += np.tril(upd[k])
            Fs = F + np.tril(F, -1).T
            L11 = np.linalg.cholesky(Fs[:s, :s])
            L21 = np.linalg.solve(L11, Fs[:s, s:]).T
            upd[i] = Fs[s:, s:] - L21 @ L21.T
            self.fronts.append((idx, L11, L21))

    def coarse_solve(self, rhs):
        cp = self.cp
        y = rhs.copy()
        for idx, L11, L21 in self.fronts:
            s = L11.shape[0]
            ys = np.linalg.solve(L11, y[idx[:s]])
            y[idx[:s]] = ys
            y[idx[s:]] -= L21 @ ys
        for idx, L11, L21 in reversed(self.fronts):
            s = L11.shape[0]
            y[idx[:s]] = np.linalg.solve(L11.T, y[idx[:s]] - L21.T @ y[idx[s:]])
        return y

    def apply(self, r):
        A = self.A
        u1 = np.zeros(self.n)
        for L in self.loc:
            fI = L["fid"][L["I"]]
            if len(fI):
                u1[fI] = np.linalg.solve(L["AII"], r[fI])
        rp = r - A @ u1
        self.dbg = dict(u1=u1.copy(), rp=rp.copy())
        ncoarse = self.cp.n if self.cp is not None else 0
        crhs = np.zeros(ncoarse)
        st = []
        for L in self.loc:
            g = L["gam"]
            rho = np.where(g >= 0, L["w"] * rp[L["fid"][L["Gn"]]], 0.0)
            u = np.linalg.solve(L["LS"].T, np.linalg.solve(L["LS"], rho))
            t = L["C"] @ u
            q = L["c"] * (L["Phi"].T @ rho)
            np.add.at(crhs, L["cc"], q)
            st.append((u, t))
        csol = self.coarse_solve(crhs) if ncoarse else crhs
        self.dbg.update(crhs=crhs.copy(), csol=csol.copy(), st=st)
        z = np.zeros(self.n)
        for L, (u, t) in zip(self.loc, st):
            e = L["c"] * csol[L["cc"]] - t
            w = L["w"] * (u + L["Phi"] @ e)
            f = L["fid"][L["Gn"]]
            ok = f >= 0
            np.add.at(z, f[ok], w[ok])
        y = r - A @ z
        for L in self.loc:
            fI = L["fid"][L["I"]]
            if len(fI):
                z[fI] = np.linalg.solve(L["AII"], y[fI])
        return z
