"""Host symbolic analysis of the coarse problem (the "analyze" phase of its factorization).

The reference factors the coarse matrix with SuperLU after a minimum-degree ordering
(bddc.py:494-511, linalg.py:117-138). On the device it is factored by a multifrontal
Cholesky; this module computes, from the constraint → owner-subdomain incidence alone
(no numbers), the geometric nested-dissection tree over the subdomain lattice, the
elimination order, every front's row structure, the extend-add maps, and the map from
local coarse blocks to the lower-triangular CSR of S_0 and from CSR entries to fronts.

ND rule: recursively halve the lattice box along its longest axis; the constraints whose
owners straddle the cut form the separator (a front); the others go to the half boxes.
Two coarse dofs couple iff they share an owner subdomain, so a subtree's boundary is
exactly the set of ancestor dofs owned by a subdomain inside the subtree's box.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class CoarsePlan:
    n: int
    perm: np.ndarray          # elimination position -> coarse id
    iperm: np.ndarray         # coarse id -> elimination position
    sep_start: np.ndarray     # per node (children before parents)
    sep_size: np.ndarray
    level: np.ndarray
    parent: np.ndarray
    bnd_ptr: np.ndarray
    bnd_idx: np.ndarray       # elimination positions, ascending per node
    rmap: np.ndarray          # position of each bnd entry in the parent's front
    # lower CSR of S_0 in elimination order (+ contributions from local blocks)
    csr_row: np.ndarray
    csr_col: np.ndarray
    csr_node: np.ndarray
    csr_frow: np.ndarray
    csr_fcol: np.ndarray
    seg_ptr: np.ndarray
    contrib: np.ndarray

    @property
    def nnodes(self) -> int:
        return len(self.sep_start)

    def front_sizes(self) -> np.ndarray:
        return self.sep_size + np.diff(self.bnd_ptr)

    def factor_flops(self) -> float:
        """Dense partial-Cholesky flops of all fronts: s^3/3 + s^2 b + s b^2."""
        s = self.sep_size.astype(float)
        b = np.diff(self.bnd_ptr).astype(float)
        return float(np.sum(s**3 / 3 + s**2 * b + s * b**2))

    def factor_entries(self) -> int:
        s = self.sep_size.astype(np.int64)
        b = np.diff(self.bnd_ptr).astype(np.int64)
        return int(np.sum(s * (s + 1) // 2 + s * b))


def _csr_from_pairs(keys: np.ndarray, vals: np.ndarray, n_keys: int):
    order = np.argsort(keys, kind="stable")
    k = keys[order]
    cnt = np.bincount(k, minlength=n_keys)
    ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    return ptr, vals[order]


def nested_dissection(owners: np.ndarray, sub_coords: np.ndarray, subs: tuple):
    """Elimination order + tree. owners: (n, W) −1-padded owner subdomains per coarse dof."""
    n = owners.shape[0]
    dim = sub_coords.shape[1]
    valid = owners >= 0
    oc = sub_coords[np.maximum(owners, 0)]  # (n, W, dim)
    big = np.iinfo(np.int64).max
    lo = np.where(valid[:, :, None], oc, big).min(axis=1)
    hi = np.where(valid[:, :, None], oc, -1).max(axis=1)

    nodes = []  # (sep dofs, children ids)
    order = []

    def rec(blo, bhi, idx):
        if len(idx) == 0:
            return None
        ext = bhi - blo
        if np.prod(ext) <= 1:
            nodes.append((np.sort(idx), []))
            return len(nodes) - 1
        ax = int(np.argmax(ext))
        mid = blo[ax] + ext[ax] // 2
        l_ax, h_ax = lo[idx, ax], hi[idx, ax]
        left = idx[h_ax < mid]
        right = idx[l_ax >= mid]
        sep = idx[(l_ax < mid) & (h_ax >= mid)]
        lhi = bhi.copy()
        lhi[ax] = mid
        rlo = blo.copy()
        rlo[ax] = mid
        kids = [c for c in (rec(blo, lhi, left), rec(rlo, bhi, right)) if c is not None]
        if len(sep) == 0 and len(kids) == 1:
            return kids[0]
        nodes.append((np.sort(sep), kids))
        return len(nodes) - 1

    root = rec(np.zeros(dim, dtype=np.int64), np.asarray(subs, dtype=np.int64),
               np.arange(n, dtype=np.int64))
    return nodes, root, lo, hi


def analyze(n: int, owners: np.ndarray, sub_coords: np.ndarray, subs: tuple,
            local_cons: list | None = None, nc_pad: int = 0,
            sub_con_ptr: np.ndarray | None = None, sub_con_ids: np.ndarray | None = None
            ) -> CoarsePlan:
    """Full symbolic analysis.

    owners     (n, W) owner subdomains of every coarse dof (constraint), −1 padded
    sub_con_ptr / sub_con_ids: CSR subdomain → its constraints in local order (coarse ids)
    """
    nodes, root, _, _ = nested_dissection(owners, sub_coords, subs)
    N = len(nodes)
    # nodes were appended in postorder (children before parents) by construction
    sep_size = np.array([len(s) for s, _ in nodes], dtype=np.int64)
    sep_start = np.concatenate([[0], np.cumsum(sep_size)[:-1]]).astype(np.int64)
    perm = np.concatenate([s for s, _ in nodes]).astype(np.int64) if N else np.zeros(0, np.int64)
    if len(perm) != n:
        raise AssertionError("nested dissection lost coarse dofs")
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    parent = -np.ones(N, dtype=np.int64)
    level = np.zeros(N, dtype=np.int64)
    for i, (_, kids) in enumerate(nodes):
        for k in kids:
            parent[k] = i
            level[i] = max(level[i], level[k] + 1)
    node_of_pos = np.repeat(np.arange(N), sep_size)

    # boundary structures, bottom-up
    bnd = [None] * N
    for i, (sep, kids) in enumerate(nodes):
        end = sep_start[i] + sep_size[i]
        own = owners[sep]
        own = np.unique(own[own >= 0])
        parts = [iperm[sub_con_ids[sub_con_ptr[p]:sub_con_ptr[p + 1]]] for p in own]
        parts += [bnd[k] for k in kids]
        cand = np.unique(np.concatenate(parts)) if parts else np.zeros(0, np.int64)
        bnd[i] = cand[cand >= end]
    bnd_ptr = np.concatenate([[0], np.cumsum([len(b) for b in bnd])]).astype(np.int64)
    bnd_idx = np.concatenate(bnd).astype(np.int64) if N else np.zeros(0, np.int64)
    rmap = np.zeros(len(bnd_idx), dtype=np.int64)
    for i in range(N):
        p = parent[i]
        if p < 0:
            if len(bnd[i]):
                raise AssertionError("root front has a boundary")
            continue
        front = np.concatenate([np.arange(sep_start[p], sep_start[p] + sep_size[p]), bnd[p]])
        pos = np.searchsorted(front, bnd[i])
        if np.any(pos >= len(front)) or np.any(front[np.minimum(pos, len(front) - 1)] != bnd[i]):
            raise AssertionError("child boundary not contained in parent front")
        rmap[bnd_ptr[i]:bnd_ptr[i + 1]] = pos
    plan = CoarsePlan(n, perm, iperm, sep_start, sep_size, level, parent, bnd_ptr, bnd_idx, rmap,
                      *([np.zeros(0, np.int64)] * 7))
    return plan


def coarse_csr(plan: CoarsePlan, sub_con_ptr: np.ndarray, sub_con_ids: np.ndarray,
               nc_pad: int) -> None:
    """Lower CSR pattern of S_0 (elimination order), segmented contribution lists and the
    CSR → front position map; stored into ``plan``.

    Local block entry (k, l) of subdomain p (col-major nc_pad × nc_pad) contributes to
    S_0[perm⁻¹ of its coarse ids]; contributions are kept in ascending-subdomain order,
    the reference's summation order (COO → CSR duplicates, bddc.py:494-504).
    """
    nsub = len(sub_con_ptr) - 1
    counts = np.diff(sub_con_ptr)
    rows, cols, cidx = [], [], []
    # group subdomains with the same local count to vectorise
    for m in np.unique(counts):
        if m == 0:
            continue
        subs_m = np.flatnonzero(counts == m)
        ids = np.stack([sub_con_ids[sub_con_ptr[p]:sub_con_ptr[p] + m] for p in subs_m])
        e = plan.iperm[ids]  # (ns, m)
        kk, ll = np.meshgrid(np.arange(m), np.arange(m), indexing="ij")
        er = e[:, kk.ravel()]
        ec = e[:, ll.ravel()]
        keep = er >= ec
        base = (subs_m.astype(np.int64) * nc_pad * nc_pad)[:, None]
        ci = base + kk.ravel()[None, :] + ll.ravel()[None, :] * nc_pad
        sub_of = np.broadcast_to(subs_m[:, None], er.shape)
        rows.append(er[keep])
        cols.append(ec[keep])
        cidx.append(np.stack([sub_of[keep], ci[keep]], axis=1))
    if not rows:
        return
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    ci = np.concatenate(cidx)
    n = plan.n
    key = r * n + c
    # stable by key then by subdomain (ascending subdomain inside each entry)
    order = np.lexsort((ci[:, 0], key))
    key = key[order]
    contrib = ci[order, 1]
    newk = np.ones(len(key), dtype=bool)
    newk[1:] = key[1:] != key[:-1]
    starts = np.flatnonzero(newk)
    seg_ptr = np.append(starts, len(key)).astype(np.int64)
    ukey = key[starts]
    csr_row = ukey // n
    csr_col = ukey % n
    # front positions: column dof c is eliminated in node(c)
    node_of_pos = np.repeat(np.arange(plan.nnodes), plan.sep_size)
    nd = node_of_pos[csr_col]
    fcol = csr_col - plan.sep_start[nd]
    frow = np.empty_like(csr_row)
    in_sep = csr_row < plan.sep_start[nd] + plan.sep_size[nd]
    frow[in_sep] = csr_row[in_sep] - plan.sep_start[nd[in_sep]]
    out = np.flatnonzero(~in_sep)
    if len(out):
        o = out[np.argsort(nd[out], kind="stable")]
        ndo = nd[o]
        bounds = np.flatnonzero(np.diff(ndo)) + 1
        for grp in np.split(o, bounds):
            i = nd[grp[0]]
            b = plan.bnd_idx[plan.bnd_ptr[i]:plan.bnd_ptr[i + 1]]
            pos = np.searchsorted(b, csr_row[grp])
            if np.any(pos >= len(b)) or np.any(b[np.minimum(pos, len(b) - 1)] != csr_row[grp]):
                raise AssertionError("coarse entry outside its front")
            frow[grp] = plan.sep_size[i] + pos
    plan.csr_row, plan.csr_col, plan.csr_node = csr_row, csr_col, nd
    plan.csr_frow, plan.csr_fcol = frow, fcol
    plan.seg_ptr, plan.contrib = seg_ptr, contrib


def coarse_csr_native(plan: CoarsePlan, sub_con_ptr: np.ndarray, sub_con_ids: np.ndarray,
                      nc_pad: int) -> None:
    """coarse_csr through the native library (csrc/host_plan.cu, bddc_coarse_pattern): the same
    arrays, O(contributions) on the host threads instead of a global lexsort."""
    import ctypes as C

    from . import _capi

    lib = _capi.load()
    i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731
    ptr, ids = i64(sub_con_ptr), i64(sub_con_ids)
    m = np.diff(ptr)
    cap = int(np.sum(m * (m + 1) // 2))
    out = {k: np.empty(max(cap, 1), dtype=np.int64) for k in ("row", "col", "node", "frow", "fcol")}
    seg = np.empty(cap + 1, dtype=np.int64)
    contrib = np.empty(max(cap, 1), dtype=np.int32)
    P = lambda a: _capi.ptr(a, C.c_longlong)  # noqa: E731
    iperm, ss, sz = i64(plan.iperm), i64(plan.sep_start), i64(plan.sep_size)
    bp, bi = i64(plan.bnd_ptr), i64(plan.bnd_idx)
    nnz = lib.bddc_coarse_pattern(len(ptr) - 1, P(ptr), P(ids), P(iperm), plan.n, int(nc_pad), plan.nnodes,
                                  P(ss), P(sz), P(bp), P(bi), P(out["row"]), P(out["col"]), P(out["node"]),
                                  P(out["frow"]), P(out["fcol"]), P(seg), _capi.ptr(contrib, C.c_int))
    if nnz < 0:
        raise AssertionError("coarse entry outside its front")
    plan.csr_row, plan.csr_col, plan.csr_node = out["row"][:nnz], out["col"][:nnz], out["node"][:nnz]
    plan.csr_frow, plan.csr_fcol = out["frow"][:nnz], out["fcol"][:nnz]
    plan.seg_ptr = seg[: nnz + 1]
    plan.contrib = contrib[:cap].astype(np.int64)


def analyze_native(n: int, owners: np.ndarray, sub_coords: np.ndarray, subs: tuple,
                   local_cons: list | None = None, nc_pad: int = 0,
                   sub_con_ptr: np.ndarray | None = None, sub_con_ids: np.ndarray | None = None
                   ) -> CoarsePlan:
    """``analyze`` through the native library (csrc/host_plan.cu, bddc_nd_build): the same
    tree, order, boundaries and maps, without the per-node numpy work (cfg5: 6 s -> < 1 s)."""
    import ctypes as C

    from . import _capi

    lib = _capi.load()
    W = owners.shape[1] if owners.ndim == 2 else 1
    dim = sub_coords.shape[1]
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
    i64 = lambda a: np.ascontiguousarray(a, dtype=np.int64)  # noqa: E731
    own, sc, sb = i32(owners), i32(sub_coords), i32(subs)
    ptr, ids = i64(sub_con_ptr), i64(sub_con_ids)
    h = C.c_void_p()
    err = C.create_string_buffer(256)
    rc = lib.bddc_nd_build(int(n), int(W), _capi.ptr(own, C.c_int), len(sub_coords), dim, _capi.ptr(sc, C.c_int),
                           _capi.ptr(sb, C.c_int), _capi.ptr(ptr, C.c_longlong), _capi.ptr(ids, C.c_longlong),
                           C.byref(h), err, len(err))
    if rc:
        raise AssertionError(err.value.decode(errors="replace"))
    try:
        N = int(lib.bddc_nd_size(h, b"nnodes"))
        nb = int(lib.bddc_nd_size(h, b"nbnd"))
        size = {"perm": n, "sep_start": N, "sep_size": N, "level": N, "parent": N, "bnd_ptr": N + 1,
                "bnd_idx": nb, "rmap": nb}
        out = {}
        for k, m in size.items():
            a = np.empty(m, dtype=np.int64)
            if lib.bddc_nd_copy(h, k.encode(), _capi.ptr(a, C.c_longlong), m):
                raise RuntimeError(f"bddc_nd_copy {k} failed")
            out[k] = a
    finally:
        lib.bddc_nd_free(h)
    perm = out["perm"]
    iperm = np.empty(n, dtype=np.int64)
    iperm[perm] = np.arange(n)
    return CoarsePlan(n, perm, iperm, out["sep_start"], out["sep_size"], out["level"], out["parent"],
                      out["bnd_ptr"], out["bnd_idx"], out["rmap"], *([np.zeros(0, np.int64)] * 7))
