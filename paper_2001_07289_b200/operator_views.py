"""Inspectable host views of a device BDDC-SO operator.

The reference keeps every per-subdomain piece of the preconditioner as host objects
(``SubdomainOperator``, bddc.py:280-306) and the coarse problem as ``coarse_matrix`` /
``coarse_factor`` (bddc.py:309-334, 494-511). The device operator holds the numbers in
HBM (explicit block inverses, Φ on the interface rows, the multifrontal coarse factor), so
these views build the reference's attributes on demand:

* index sets (``global_dofs``, ``gamma_local``, ``coarse_ids``, ``constraint_rows`` …) from
  the host partition and constraint tables, with the reference's rules (bddc.py:419-450,
  472, 490);
* ``coarse_basis`` Ψ_i from the device's Φ_i (interface rows, Ψ = c_i Φ) — its interior rows
  are the discrete harmonic extension −A_II⁻¹A_IΓΨ_Γ (the saddle solve's interior
  stationarity), computed on the host for this one subdomain when asked for;
* ``coarse_matrix`` from the device-assembled S_0 (CSR values read back, permuted from
  elimination order to coarse ids, upper triangle as the reference stores it);
* ``coarse_factor.solve`` through the device multifrontal factor (``bddc_coarse_solve``).

They are diagnostics of the device state (tests compare them with the oracle); nothing on
the setup / apply / PCG path reads them.
"""

from __future__ import annotations

import ctypes as C
from functools import cached_property

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import _capi
from .linalg import SparseSym
from .mesh import assemble_cells


def _read(op, name: str, offset: int, count: int) -> np.ndarray:
    out = np.empty(count)
    got = op._lib.bddc_read_buffer(op._ctx, name.encode(), int(offset), int(count),
                                   _capi.ptr(out, C.c_double))
    if got != count:
        raise RuntimeError(f"reading device buffer {name}[{offset}:{offset + count}] failed")
    return out


class SubdomainView:
    """One subdomain of a device operator with the reference's SubdomainOperator fields.

    ``interior_factor`` and ``saddle`` are ``None``: on the device they exist only as explicit
    block inverses inside the packed factor buffers, not as factorization objects.
    """

    interior_factor = None
    saddle = None

    def __init__(self, op, sub: int):
        self._op = op
        self.sub_id = int(sub)

    # ---- index sets (bddc.py:419-433) ----
    @cached_property
    def _cells(self) -> np.ndarray:
        return np.flatnonzero(self._op.pair.theta == self.sub_id)

    @cached_property
    def _local_nodes(self) -> np.ndarray:
        mesh = self._op.system.mesh
        nodes = np.unique(mesh.cell_nodes[self._cells])
        return nodes[mesh.node_to_free[nodes] >= 0]

    @cached_property
    def global_dofs(self) -> np.ndarray:
        return self._op.system.mesh.node_to_free[self._local_nodes].astype(np.int64)

    @cached_property
    def _gpos(self) -> np.ndarray:
        return self._op._gamma_index[self.global_dofs]

    @cached_property
    def gamma_local(self) -> np.ndarray:
        return np.flatnonzero(self._gpos >= 0)

    @cached_property
    def interior_local(self) -> np.ndarray:
        return np.flatnonzero(self._gpos < 0)

    @property
    def gamma_global(self) -> np.ndarray:
        return self.global_dofs[self.gamma_local]

    @property
    def interior_global(self) -> np.ndarray:
        return self.global_dofs[self.interior_local]

    @property
    def gamma_positions(self) -> np.ndarray:
        return self._gpos[self.gamma_local]

    @property
    def gamma_weights(self) -> np.ndarray:
        g = self.gamma_global
        return self._op.weights.weights_for(np.full(len(g), self.sub_id), g)

    # ---- constraints (bddc.py:411-414, 441-450) ----
    @cached_property
    def coarse_ids(self) -> np.ndarray:
        cons = self._op.constraints
        own = cons.objects.owners[cons.con_obj]
        return np.flatnonzero(np.any(own == self.sub_id, axis=1)).astype(np.int64)

    @cached_property
    def constraint_rows(self) -> sp.csr_matrix:
        cons = self._op.constraints
        local = np.full(self._op.n, -1, dtype=np.int64)
        local[self.global_dofs] = np.arange(len(self.global_dofs))
        ids = self.coarse_ids
        lens = cons.dof_ptr[ids + 1] - cons.dof_ptr[ids]
        idx = np.concatenate([np.arange(cons.dof_ptr[c], cons.dof_ptr[c + 1]) for c in ids]) \
            if len(ids) else np.zeros(0, np.int64)
        rows = np.repeat(np.arange(len(ids)), lens)
        return sp.csr_matrix((cons.coeff[idx], (rows, local[cons.dof_list[idx]])),
                             shape=(len(ids), len(self.global_dofs)))

    # ---- host assemblies (bddc.py:427, 471) ----
    @cached_property
    def neumann(self) -> SparseSym:
        return assemble_cells(self._op.system.mesh, self._op.system.coeff, self._cells,
                              self._local_nodes)

    @property
    def coupling(self) -> sp.csr_matrix:
        return self.neumann.tocsr()[self.interior_local][:, self.gamma_local]

    # ---- device data ----
    @cached_property
    def coarse_basis(self) -> np.ndarray:
        """Ψ_i (n_local × n_c) = c_i Φ_i on the interface rows (device), harmonic inside."""
        op = self._op
        sl = op.slab
        if not sl.s_lo <= self.sub_id < sl.s_hi:
            raise ValueError(f"subdomain {self.sub_id} is not on this rank")
        plan = op.plan
        ng, ncp = plan.layout.nG_pad, plan.nc_pad
        nc = len(self.coarse_ids)
        phi = _read(op, "Phi", (self.sub_id - sl.s_lo) * ng * ncp, ng * ncp).reshape(ncp, ng).T
        c = _read(op, "cscale", self.sub_id, 1)[0]
        psi = np.zeros((len(self.global_dofs), nc))
        slot_g = plan.slot_gamma[self.sub_id, : plan.layout.nG]
        ok = slot_g >= 0
        local = np.full(op.n, -1, dtype=np.int64)
        local[self.global_dofs] = np.arange(len(self.global_dofs))
        rows = local[op.gamma_dofs[slot_g[ok]]]
        psi[rows] = c * phi[: plan.layout.nG][ok, :nc]
        if len(self.interior_local) and nc:
            A = self.neumann.tocsr()
            I, G = self.interior_local, self.gamma_local
            psi[I] = -spla.splu(A[I][:, I].tocsc()).solve(A[I][:, G] @ psi[G])
        return psi

    @property
    def n_local(self) -> int:
        return len(self.global_dofs)

    @property
    def n_coarse(self) -> int:
        return len(self.coarse_ids)


class SubdomainList:
    """Sequence of lazy :class:`SubdomainView` (``BddcOperator.subdomains``)."""

    def __init__(self, op):
        self._op = op
        self._cache = {}

    def __len__(self):
        return self._op.pair.subdomain_count

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        i = int(i)
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        if i not in self._cache:
            self._cache[i] = SubdomainView(self._op, i)
        return self._cache[i]

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


def device_coarse_pattern(op):
    """(row, col, seg_ptr, contrib) of the coarse assembly pattern the setup built on the
    device (elimination order; bddc_coarse_csr)."""
    import ctypes as C

    lib = op._lib
    nnz = lib.bddc_coarse_csr(op._ctx, None, None, None, None, 0, 0)
    if nnz < 0:
        raise RuntimeError("no device-built coarse pattern")
    m = sum(int(k) * (int(k) + 1) // 2 for k in op.plan.n_con_local)
    row = np.empty(nnz, np.int64)
    col = np.empty(nnz, np.int64)
    seg = np.empty(nnz + 1, np.int64)
    con = np.empty(max(m, 1), np.int32)
    P = lambda a: a.ctypes.data_as(C.POINTER(C.c_longlong))  # noqa: E731
    got = lib.bddc_coarse_csr(op._ctx, P(row), P(col), P(seg), con.ctypes.data_as(C.POINTER(C.c_int)), nnz, m)
    if got != nnz:
        raise RuntimeError("bddc_coarse_csr failed")
    return row, col, seg, con[:m].astype(np.int64)


def coarse_matrix(op) -> SparseSym | None:
    """S_0 as the reference stores it: upper triangle in coarse-id order (bddc.py:494-505),
    values from the device's deterministic segmented assembly."""
    cp = op.plan.coarse
    if cp is None:
        return None
    row, col = cp.csr_row, cp.csr_col
    if len(cp.contrib) == 0:  # pattern built on the device (coarse_pattern.cu)
        row, col, _, _ = device_coarse_pattern(op)
    val = _read(op, "csr_val", 0, len(row))
    r = cp.perm[row]
    c = cp.perm[col]
    return SparseSym.from_upper_triplets(cp.n, np.minimum(r, c), np.maximum(r, c), val)


class CoarseFactor:
    """``coarse_factor``: S_0⁻¹ through the device multifrontal factor (bddc.py:362-364)."""

    def __init__(self, op):
        self._op = op
        self.n = op.plan.coarse.n

    def solve(self, rhs):
        op = self._op
        torch = op._torch
        cp = op.plan.coarse
        b = np.asarray(rhs, dtype=np.float64)
        if b.shape != (cp.n,):
            raise ValueError(f"coarse right-hand side has shape {b.shape}, expected ({cp.n},)")
        dev = f"cuda:{op.device}"
        bd = torch.from_numpy(np.ascontiguousarray(b[cp.perm])).to(dev)
        xd = torch.empty_like(bd)
        stream = torch.cuda.current_stream(bd.device).cuda_stream
        rc = op._lib.bddc_coarse_solve(op._ctx, C.c_void_p(bd.data_ptr()), C.c_void_p(xd.data_ptr()),
                                       C.c_void_p(stream))
        if rc:
            raise RuntimeError("bddc_coarse_solve failed")
        xe = xd.cpu().numpy()
        op._check_async()
        x = np.empty(cp.n)
        x[cp.perm] = xe
        return x
