"""Host construction of the device operator's index tables (integer work, bit-exact).

Everything the CUDA setup needs besides the coefficient: the local layout shared by all
subdomains of a uniform box partition, per-subdomain interface slots with weights and
constraint membership, interface / coarse gather tables, and the coarse symbolic plan.
Reference correspondence (bddc.py:404-492):

* local dofs ascending, gamma_local / interior_local split       bddc.py:420-433
* constraint rows in coarse_id order of the constraints owned   bddc.py:411-414, 441-450
* gamma_weights aligned with gamma_global                        bddc.py:472
* gamma_positions / coarse_ids scatter targets                   bddc.py:360, 371, 490
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import symbolic
from .partition import PartitionPair
from .weights import ConstraintTable, WeightingOperator


# coarse CSR pattern: the native statement (csrc/host_plan.cu); symbolic.coarse_csr is the
# numpy statement it is checked against (tests/test_host_plan.py)
COARSE_CSR = symbolic.coarse_csr_native
# ND analysis: the native statement (host_plan.cu); symbolic.analyze is its numpy checker
ANALYZE = symbolic.analyze_native


def _round(x: int, m: int) -> int:
    return (x + m - 1) // m * m


@dataclass
class LocalLayout:
    dim: int
    blk: tuple
    nloc_nodes: int
    nG: int
    nG_pad: int
    m: int
    m_pad: int
    nblk: int
    nI_pad: int
    node_code: np.ndarray   # >=0 interior row j*m_pad + r; <0 −(slot+1)
    slot_node: np.ndarray   # [nG]
    irow_node: np.ndarray   # [nI_pad], −1 on padding
    slot_coords: np.ndarray  # [nG, dim] local node coordinates


def local_layout(dim: int, blk: tuple) -> LocalLayout:
    npd = [b + 1 for b in blk]
    nloc = int(np.prod(npd))
    ids = np.arange(nloc)
    coords = np.zeros((nloc, dim), dtype=np.int64)
    rem = ids.copy()
    for d in range(dim):
        coords[:, d] = rem % npd[d]
        rem //= npd[d]
    interior = np.all((coords >= 1) & (coords <= np.asarray(blk) - 1), axis=1)
    m = int(np.prod([b - 1 for b in blk[:-1]]))
    nblk = blk[-1] - 1
    m_pad = _round(max(m, 1), 8)
    nI_pad = m_pad * max(nblk, 0)
    code = np.zeros(nloc, dtype=np.int32)
    # interior row: plane j = last coord − 1, row r = x-fastest index over the other coords
    r = np.zeros(nloc, dtype=np.int64)
    st = 1
    for d in range(dim - 1):
        r += (coords[:, d] - 1) * st
        st *= blk[d] - 1
    j = coords[:, dim - 1] - 1
    row = j * m_pad + r
    code[interior] = row[interior]
    surf = np.flatnonzero(~interior)
    code[surf] = -(np.arange(len(surf)) + 1)
    nG = len(surf)
    irow = -np.ones(nI_pad, dtype=np.int32)
    irow[row[interior]] = np.flatnonzero(interior)
    return LocalLayout(dim, tuple(blk), nloc, nG, _round(nG, 8), m, m_pad, max(nblk, 0), nI_pad,
                       code, surf.astype(np.int32), irow, coords[surf])


@dataclass
class DevicePlan:
    layout: LocalLayout
    nsub: int
    nc_pad: int
    slot_gamma: np.ndarray
    slot_w: np.ndarray
    slot_con: np.ndarray
    slot_coef: np.ndarray
    con_coarse: np.ndarray
    gamma_dof: np.ndarray
    gamma_slots: np.ndarray
    coarse_slots: np.ndarray
    coarse: symbolic.CoarsePlan | None
    n_con_local: np.ndarray


def build_device_plan(pair: PartitionPair, cons: ConstraintTable,
                      weights: WeightingOperator, coarse_pattern: str = "host",
                      device: int | None = None) -> DevicePlan:
    """``coarse_pattern``: "host" computes the coarse assembly pattern here (symbolic.py /
    host_plan.cu); "device" leaves it to the setup, which builds it on the GPU from
    ``con_coarse`` (coarse_pattern.cu). ``device`` (CUDA ordinal): the per-subdomain slot
    tables and the interface gather table come from the device kernels (index_sets.cu,
    bddc_layout_tables), bit-identical to the numpy statement below."""
    mesh = pair.mesh
    layout_info = pair.box_layout
    if layout_info is None:
        raise ValueError("the device operator needs a uniform box partition (partition_uniform)")
    subs, blk = layout_info
    dim = mesh.dim
    lay = local_layout(dim, blk)
    nsub = int(np.prod(subs))
    W = 2**dim
    objects = cons.objects
    ms = pair.membership
    gamma = ms.gamma_dofs
    nfree = mesh.free_count
    gidx = -np.ones(nfree, dtype=np.int64)
    gidx[gamma] = np.arange(len(gamma))

    # subdomain lattice coordinates (x-fastest ids, partition.py:146-153)
    pid = np.arange(nsub)
    pc = np.zeros((nsub, dim), dtype=np.int64)
    rem = pid.copy()
    for d in range(dim):
        pc[:, d] = rem % subs[d]
        rem //= subs[d]

    cells = np.asarray(mesh.cells_per_dim)
    nf = cells - 1
    nG, nG_pad = lay.nG, lay.nG_pad
    if device is None:
        # global free dof of every (sub, slot)
        gcoords = pc[:, None, :] * np.asarray(blk)[None, None, :] + lay.slot_coords[None, :, :]
        dirichlet = np.any((gcoords == 0) | (gcoords == cells), axis=2)
        fid = np.zeros(gcoords.shape[:2], dtype=np.int64)
        st = 1
        for d in range(dim):
            fid += (gcoords[:, :, d] - 1) * st
            st *= int(nf[d])
        fid[dirichlet] = -1

    # constraint of each free dof
    n_con = len(cons)
    con_of = -np.ones(nfree, dtype=np.int64)
    coef_of = np.zeros(nfree)
    cnt = np.diff(cons.dof_ptr)
    con_of[cons.dof_list] = np.repeat(np.arange(n_con), cnt)
    coef_of[cons.dof_list] = cons.coeff

    # local constraint numbering: constraints owned by p in coarse-id order
    con_owners = objects.owners[cons.con_obj] if n_con else np.zeros((0, W), np.int64)
    pv = con_owners >= 0
    pair_sub = con_owners[pv]
    pair_con = np.broadcast_to(np.arange(n_con)[:, None], con_owners.shape)[pv]
    order = np.lexsort((pair_con, pair_sub))
    pair_sub, pair_con = pair_sub[order], pair_con[order]
    n_local = np.bincount(pair_sub, minlength=nsub)
    sub_con_ptr = np.concatenate([[0], np.cumsum(n_local)]).astype(np.int64)
    local_k = np.arange(len(pair_sub)) - sub_con_ptr[pair_sub]
    nc_max = int(n_local.max()) if nsub else 0
    nc_pad = _round(max(nc_max, 1), 8)
    pair_key = pair_sub * max(n_con, 1) + pair_con

    def lookup_k(sub, con):
        key = sub * max(n_con, 1) + con
        pos = np.searchsorted(pair_key, key)
        return local_k[pos]

    if device is not None:
        dev_tables = _device_slot_tables(device, pair, lay, subs, nsub, nG_pad, gamma, con_of, coef_of,
                                         objects, weights, sub_con_ptr, pair_con)
    if device is None:
        valid = fid >= 0
        slot_gamma = -np.ones((nsub, nG_pad), dtype=np.int32)
    if device is None:
        slot_w = np.zeros((nsub, nG_pad))
        slot_con = -np.ones((nsub, nG_pad), dtype=np.int32)
        slot_coef = np.zeros((nsub, nG_pad))
        sub_idx = np.broadcast_to(pid[:, None], fid.shape)
        fv = fid[valid]
        sv = sub_idx[valid]
        sg = slot_gamma[:, :nG]
        sg[valid] = gidx[fv]
        if np.any(gidx[fv] < 0):
            raise AssertionError("a free surface node is not on the interface")
        slot_gamma[:, :nG] = sg
        cv = con_of[fv]
        has = cv >= 0
        sc = slot_con[:, :nG]
        tmp = -np.ones(len(fv), dtype=np.int64)
        tmp[has] = lookup_k(sv[has], cv[has])
        sc[valid] = tmp
        slot_con[:, :nG] = sc
        sco = slot_coef[:, :nG]
        sco[valid] = np.where(has, coef_of[fv], 0.0)
        slot_coef[:, :nG] = sco
    else:
        slot_gamma, slot_con, slot_coef, slot_w, gamma_slots_dev = dev_tables

    # coarse plan (elimination order) and the constraint maps
    plan = None
    con_coarse = -np.ones((nsub, nc_pad), dtype=np.int32)
    coarse_slots = -np.ones((max(n_con, 0), W), dtype=np.int32)
    if n_con:
        plan = ANALYZE(n_con, con_owners, pc, tuple(subs), sub_con_ptr=sub_con_ptr,
                                sub_con_ids=pair_con)
        if coarse_pattern == "host":
            COARSE_CSR(plan, sub_con_ptr, pair_con, nc_pad)
        con_coarse[pair_sub, local_k] = plan.iperm[pair_con]
        # owners of each constraint (ascending) -> slot sub*nc_pad + k, rows in elimination order
        ks = np.where(pv, 0, -1).astype(np.int64)
        ks[pv] = lookup_k(con_owners[pv], np.broadcast_to(np.arange(n_con)[:, None], con_owners.shape)[pv])
        slots = np.where(pv, con_owners * nc_pad + ks, -1)
        coarse_slots = slots[plan.perm].astype(np.int32)

    # interface gather: owner slots of each gamma dof, ascending subdomain
    if device is not None:
        dp = DevicePlan(lay, nsub, nc_pad, slot_gamma, slot_w, slot_con, slot_coef, con_coarse,
                        gamma.astype(np.int64), gamma_slots_dev, coarse_slots, plan, n_local)
        return dp
    gobj = objects.dof_obj[gamma]
    gown = objects.owners[gobj]  # (n_gamma, W) ascending, −1 padded
    gv = gown >= 0
    gcoord = np.zeros((len(gamma), dim), dtype=np.int64)
    rem = gamma.copy()
    for d in range(dim):
        gcoord[:, d] = rem % nf[d] + 1
        rem //= nf[d]
    slot_of_node = np.full(lay.nloc_nodes, -1, dtype=np.int64)
    slot_of_node[lay.slot_node] = np.arange(nG)
    npd = np.asarray(blk) + 1
    loc = gcoord[:, None, :] - pc[np.maximum(gown, 0)] * np.asarray(blk)[None, None, :]
    lnode = np.zeros(gown.shape, dtype=np.int64)
    st = 1
    for d in range(dim):
        lnode += loc[:, :, d] * st
        st *= int(npd[d])
    sl = slot_of_node[np.where(gv, lnode, 0)]
    if np.any(gv & (sl < 0)):
        raise AssertionError("interface dof does not map to a surface slot")
    gamma_slots = np.where(gv, gown * nG_pad + sl, -1).astype(np.int32)

    dp = DevicePlan(lay, nsub, nc_pad, slot_gamma, slot_w, slot_con, slot_coef, con_coarse,
                    gamma.astype(np.int64), gamma_slots, coarse_slots, plan, n_local)
    dp.slot_w = slot_weights(dp, weights)
    return dp


def slot_weights(plan: DevicePlan, weights: WeightingOperator) -> np.ndarray:
    """[nsub, nG_pad] weight δ†_i of every interface slot (bddc.py:472), 0 on Dirichlet /
    padding slots; recomputed when a new α changes coefficient weights (refactor)."""
    sg = plan.slot_gamma
    valid = sg >= 0
    sub = np.broadcast_to(np.arange(plan.nsub)[:, None], sg.shape)[valid]
    out = np.zeros(sg.shape)
    out[valid] = weights.weights_for(sub, plan.gamma_dof[sg[valid]])
    return out


def _device_slot_tables(device, pair, lay, subs, nsub, nG_pad, gamma, con_of, coef_of, objects, weights,
                        sub_con_ptr, pair_con):
    """slot_gamma / slot_con / slot_coef / slot_w [nsub, nG_pad] and gamma_slots [n_gamma, 2^d]
    from the device kernels (bddc_layout_tables)."""
    import ctypes as C

    from . import _capi

    lib = _capi.load()
    mesh = pair.mesh
    dim = mesh.dim
    W = 2**dim
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
    f64 = lambda a: np.ascontiguousarray(a, dtype=np.float64)  # noqa: E731
    cells = i32(list(mesh.cells_per_dim) + [1] * (3 - dim))
    subs3 = i32(list(subs) + [1] * (3 - dim))
    slot_of_node = np.full(lay.nloc_nodes, -1, dtype=np.int32)
    slot_of_node[lay.slot_node] = np.arange(lay.nG, dtype=np.int32)
    args = dict(sc=i32(lay.slot_coords), son=slot_of_node, gamma=i32(gamma), con=i32(con_of), coef=f64(coef_of),
                dobj=i32(objects.dof_obj), own=i32(objects.owners), w=f64(weights.obj_weights),
                ptr=np.ascontiguousarray(sub_con_ptr, dtype=np.int64), scon=i32(pair_con))
    out_sg = np.empty((nsub, nG_pad), np.int32)
    out_sc = np.empty((nsub, nG_pad), np.int32)
    out_co = np.empty((nsub, nG_pad), np.float64)
    out_w = np.empty((nsub, nG_pad), np.float64)
    out_gs = np.empty((len(gamma), W), np.int32)
    pi, pd, pll = C.c_int, C.c_double, C.c_longlong
    P = _capi.ptr
    err = C.create_string_buffer(512)
    rc = lib.bddc_layout_tables(int(device), dim, P(cells, pi), P(subs3, pi), lay.nG, nG_pad, lay.nloc_nodes,
                                P(args["sc"], pi), P(args["son"], pi), mesh.free_count, P(args["gamma"], pi),
                                len(gamma), P(args["con"], pi), P(args["coef"], pd), P(args["dobj"], pi),
                                len(objects), P(args["own"], pi), P(args["w"], pd), P(args["ptr"], pll),
                                P(args["scon"], pi), P(out_sg, pi), P(out_sc, pi), P(out_co, pd), P(out_w, pd),
                                P(out_gs, pi), err, len(err))
    if rc:
        raise RuntimeError("device layout tables: " + err.value.decode(errors="replace"))
    if np.any(out_gs == -2):
        raise AssertionError("interface dof does not map to a surface slot")
    return out_sg, out_sc, out_co, out_w, out_gs
