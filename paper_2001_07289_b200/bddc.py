"""BDDC-SO operator on the GPU: ``build_bddc`` / ``BddcOperator.apply`` drop-in.

Mirrors ``bddcso.bddc`` (reference ``pkg/src/bddcso/bddc.py``). Host index sets (weights,
constraints, sufficiency) come from :mod:`.weights` (bit-exact with bddc.py:108-277); the
numeric setup (bddc.py:393-523) and the apply (bddc.py:336-390) run as sm_100a CUDA
through the C ABI of ``include/bddcso_b200.h``.

Extension (documented in DESIGN.md): ``coarse_scaling`` = "reference" reproduces the
reference's coarse basis Ψ_i = Φ_i / s_i² (linalg.py:165-171 with bddc.py:457); "spec"
gives the documented C Ψ = I.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _capi
from . import operator_views
from .layout import DevicePlan, build_device_plan, slot_weights
from .linalg import NotSpdError, UnderconstrainedError
from .mesh import AssembledSystem, CoefficientField, element_matrix_box
from .partition import ObjectTable, PartitionPair
from .shard import slab_ranges
from .weights import (ConstraintTable, Recipe, RecipeError, WeightingOperator,
                      compute_weights, select_constraints)

COARSE_SCALINGS = ("reference", "spec")


class NotSpdOperatorError(ValueError):
    """An inner product required to be positive is not (krylov.py:12)."""


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("the BDDC-SO device operator needs a CUDA GPU (no CPU fallback)")
    return torch


def raise_for(code: int, msg: str, recipe=None):
    if code == 0:
        return
    if code == 1:
        raise ValueError(msg or "invalid argument")
    if code == 2:
        raise NotSpdError(msg)
    if code == 3:
        raise UnderconstrainedError(msg)
    if code == 4:
        raise NotSpdError(f"coarse matrix not SPD; recipe {recipe} is insufficient: {msg}")
    if code == 5:
        raise NotSpdOperatorError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


@dataclass
class SetupTimes:
    prep_s: float = 0.0       # host index tables + symbolic analysis
    upload_ms: float = 0.0    # host -> device of the descriptor
    local_ms: float = 0.0     # batched subdomain factorizations (CUDA events)
    coarse_ms: float = 0.0    # coarse assembly + multifrontal factorization (CUDA events)


class BddcOperator:
    """Two-level BDDC(-SO) preconditioner held on the GPU (bddc.py:309-390)."""

    def __init__(self, system: AssembledSystem, pair: PartitionPair, weights: WeightingOperator,
                 recipe: Recipe, constraints: ConstraintTable, plan: DevicePlan,
                 coarse_scaling: str = "reference", device: int = 0, comm=None):
        self.system = system
        self.pair = pair
        self.weights = weights
        self.recipe = recipe
        self.constraints = constraints
        self.coarse_size = len(constraints)
        self.gamma_dofs = pair.membership.gamma_dofs
        self.plan = plan
        self.coarse_scaling = coarse_scaling
        self.device = device
        self.n = system.mesh.free_count
        self.times = SetupTimes()
        self._lib = _capi.load()
        self._torch = _torch()
        self._ctx = C.c_void_p()
        rc = self._lib.bddc_create(device, C.byref(self._ctx))
        if rc:
            raise RuntimeError(f"bddc_create failed ({rc})")
        # multi-GPU (shard.py): this rank's slab; vectors stay global-length, inputs valid on
        # the active rows, outputs on the owned rows
        self.comm = comm
        rank, world = (comm.rank, comm.world) if comm is not None else (0, 1)
        mesh = system.mesh
        self.slab = slab_ranges(mesh.dim, mesh.cells_per_dim, pair.box_layout[0], rank, world)
        if comm is not None:
            comm.attach(self._lib, self._ctx)
        self._desc_arrays = None
        self._desc = None

    # ------------------------------------------------ reference attributes (views)
    @property
    def subdomains(self) -> operator_views.SubdomainList:
        """Per-subdomain pieces (bddc.py:280-306), built lazily from the host tables and the
        device buffers (operator_views.py)."""
        if getattr(self, "_subdomains", None) is None:
            self._subdomains = operator_views.SubdomainList(self)
        return self._subdomains

    @property
    def coarse_matrix(self):
        """S_0 (SparseSym, upper triangle, coarse-id order) from the device assembly."""
        return operator_views.coarse_matrix(self)

    @property
    def coarse_factor(self):
        """Object with ``solve(rhs)`` running the device coarse factor (None without a coarse
        space, as the reference's)."""
        return operator_views.CoarseFactor(self) if self.plan.coarse is not None else None

    @property
    def _gamma_index(self) -> np.ndarray:
        gi = getattr(self, "_gidx", None)
        if gi is None:
            gi = np.full(self.n, -1, dtype=np.int64)
            gi[self.gamma_dofs] = np.arange(len(self.gamma_dofs))
            self._gidx = gi
        return gi

    # ---------------------------------------------------------------- setup
    def _descriptor(self):
        p = self.plan
        lay = p.layout
        mesh = self.system.mesh
        dim = mesh.dim
        arrs = {}

        def keep(name, a, dtype):
            a = np.ascontiguousarray(a, dtype=dtype)
            arrs[name] = a
            return a

        d = _capi.SetupDesc()
        d.dim = dim
        for k in range(3):
            d.cells[k] = mesh.cells_per_dim[k] if k < dim else 1
            d.subs[k] = self.pair.box_layout[0][k] if k < dim else 1
        d.element = 1 if mesh.element == "p1" else 0
        d.coarse_scaling = COARSE_SCALINGS.index(self.coarse_scaling)
        d.alpha = _capi.ptr(keep("alpha", self.system.coeff.alpha, np.float64), C.c_double)
        K = element_matrix_box(mesh.spacings, mesh.element)
        d.elem_K = _capi.ptr(keep("K", K.ravel(), np.float64), C.c_double)
        d.nloc_nodes, d.nG, d.nG_pad = lay.nloc_nodes, lay.nG, lay.nG_pad
        d.m, d.m_pad, d.nblk, d.nI_pad, d.nc_pad = lay.m, lay.m_pad, lay.nblk, lay.nI_pad, p.nc_pad
        i32, i64, f64 = C.c_int, C.c_longlong, C.c_double
        d.node_code = _capi.ptr(keep("node_code", lay.node_code, np.int32), i32)
        d.slot_node = _capi.ptr(keep("slot_node", lay.slot_node, np.int32), i32)
        d.irow_node = _capi.ptr(keep("irow_node", lay.irow_node, np.int32), i32)
        d.slot_gamma = _capi.ptr(keep("slot_gamma", p.slot_gamma, np.int32), i32)
        d.slot_w = _capi.ptr(keep("slot_w", p.slot_w, np.float64), f64)
        d.slot_con = _capi.ptr(keep("slot_con", p.slot_con, np.int32), i32)
        d.slot_coef = _capi.ptr(keep("slot_coef", p.slot_coef, np.float64), f64)
        d.con_coarse = _capi.ptr(keep("con_coarse", p.con_coarse, np.int32), i32)
        d.n_gamma = len(p.gamma_dof)
        d.gamma_dof = _capi.ptr(keep("gamma_dof", p.gamma_dof, np.int64), i64)
        d.gamma_slots = _capi.ptr(keep("gamma_slots", p.gamma_slots, np.int32), i32)
        cp = p.coarse
        d.n_coarse = self.coarse_size
        d.coarse_slots = _capi.ptr(keep("coarse_slots", p.coarse_slots, np.int32), i32)
        if cp is not None:
            d.nnodes = cp.nnodes
            d.node_sep_start = _capi.ptr(keep("sep_start", cp.sep_start, np.int32), i32)
            d.node_sep_size = _capi.ptr(keep("sep_size", cp.sep_size, np.int32), i32)
            d.node_level = _capi.ptr(keep("level", cp.level, np.int32), i32)
            d.node_parent = _capi.ptr(keep("parent", cp.parent, np.int32), i32)
            d.bnd_ptr = _capi.ptr(keep("bnd_ptr", cp.bnd_ptr, np.int32), i32)
            d.bnd_idx = _capi.ptr(keep("bnd_idx", cp.bnd_idx, np.int32), i32)
            d.rmap = _capi.ptr(keep("rmap", cp.rmap, np.int32), i32)
            if len(cp.contrib):  # host-built assembly pattern (else built on the device)
                d.nnz = len(cp.csr_row)
                d.csr_node = _capi.ptr(keep("csr_node", cp.csr_node, np.int32), i32)
                d.csr_row = _capi.ptr(keep("csr_frow", cp.csr_frow, np.int32), i32)
                d.csr_col = _capi.ptr(keep("csr_fcol", cp.csr_fcol, np.int32), i32)
                d.seg_ptr = _capi.ptr(keep("seg_ptr", cp.seg_ptr, np.int64), i64)
                d.ncontrib = len(cp.contrib)
                d.contrib = _capi.ptr(keep("contrib", cp.contrib, np.int32), i32)
        self._desc_arrays = arrs
        self._desc = d
        return d

    def _setup(self):
        d = self._descriptor()
        err = C.create_string_buffer(1024)
        rc = self._lib.bddc_setup(self._ctx, C.byref(d), err, len(err))
        self.setup_code = rc
        if rc and os.environ.get("BDDC_DEBUG_KEEP"):
            return
        raise_for(rc, err.value.decode(errors="replace"), self.recipe)
        self._read_times()

    def refactor(self, alpha: np.ndarray | None = None):
        """Re-run the numeric setup on device-resident inputs, optionally for a new α on the
        same partition. With coefficient weighting (Remark 1, bddc.py:108-145) the interface
        weights depend on α: they are recomputed on the host and uploaded before the setup,
        so the result is the reference's build_bddc for the new coefficient. ``system`` is
        replaced by the new-α system (its host matrix, if ever needed, is rebuilt lazily)."""
        err = C.create_string_buffer(1024)
        a = None
        if alpha is not None:
            coeff = CoefficientField(np.ascontiguousarray(alpha, dtype=np.float64))
            if coeff.alpha.shape != (self.system.mesh.cell_count,):
                raise ValueError(f"alpha has shape {coeff.alpha.shape}, expected "
                                 f"({self.system.mesh.cell_count},)")
            a = coeff.alpha
            if self.weights.mode == "coefficient":
                weights = compute_weights(self.pair, "coefficient", coeff, self.weights.objects)
                slot_w = np.ascontiguousarray(slot_weights(self.plan, weights))
                rc = self._lib.bddc_update_weights(self._ctx, _capi.ptr(slot_w, C.c_double), err, len(err))
                raise_for(rc, err.value.decode(errors="replace"), self.recipe)
                self.weights = weights
            self.system = AssembledSystem(self.system.mesh, coeff, self.system.rhs)
        rc = self._lib.bddc_refactor(self._ctx, _capi.ptr(a, C.c_double) if a is not None else None,
                                     err, len(err))
        raise_for(rc, err.value.decode(errors="replace"), self.recipe)
        self._read_times()

    def _read_times(self):
        st = self.stats()
        self.times.upload_ms = st.t_upload_ms
        self.times.local_ms = st.t_local_ms
        self.times.coarse_ms = st.t_coarse_ms

    def stats(self) -> _capi.Stats:
        st = _capi.Stats()
        self._lib.bddc_get_stats(self._ctx, C.byref(st))
        return st

    # ---------------------------------------------------------------- apply
    def _as_device(self, v, name: str = "vector", n: int | None = None):
        """(device tensor, came-in-as-tensor). CUDA tensors must already be float64, of shape
        (n,), contiguous and on this operator's device: the C ABI reads / writes exactly n
        doubles, so anything else is rejected instead of converted behind the caller's back.
        Host arrays (numpy / lists / CPU tensors) are copied to the device."""
        torch = self._torch
        n = self.n if n is None else n
        if isinstance(v, torch.Tensor) and v.device.type == "cuda":
            if v.dtype != torch.float64:
                raise ValueError(f"{name} must be float64, got {v.dtype}")
            if tuple(v.shape) != (n,):
                raise ValueError(f"{name} has shape {tuple(v.shape)}, expected ({n},)")
            if v.device.index != self.device:
                raise ValueError(f"{name} is on {v.device}, the operator on cuda:{self.device}")
            if not v.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
            return v, True
        a = np.asarray(v.cpu().numpy() if isinstance(v, torch.Tensor) else v, dtype=np.float64)
        if a.shape != (n,):
            raise ValueError(f"{name} has shape {a.shape}, expected ({n},)")
        return torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{self.device}"), False

    def _check_async(self):
        """Raise if the last apply failed asynchronously (coarse-solve dependency timeout)."""
        err = C.create_string_buffer(512)
        rc = self._lib.bddc_check(self._ctx, err, len(err))
        raise_for(rc, err.value.decode(errors="replace"))

    def apply(self, r):
        """z = B r (bddc.py:336-380). numpy in → numpy out; CUDA tensor in → CUDA tensor out."""
        torch = self._torch
        if tuple(np.shape(r)) != (self.n,):
            raise ValueError(f"residual has shape {tuple(np.shape(r))}, expected ({self.n},)")
        rd, is_tensor = self._as_device(r, "residual")
        z = torch.empty_like(rd)
        stream = torch.cuda.current_stream(rd.device).cuda_stream
        rc = self._lib.bddc_apply(self._ctx, C.c_void_p(rd.data_ptr()), C.c_void_p(z.data_ptr()),
                                  C.c_void_p(stream))
        raise_for(rc, "bddc_apply failed")
        if is_tensor:
            return z
        out = z.cpu().numpy()
        self._check_async()
        return out

    __call__ = apply

    def matvec(self, x):
        """A x (matrix-free, the system operator of this preconditioner)."""
        torch = self._torch
        xd, is_tensor = self._as_device(x, "x")
        y = torch.empty_like(xd)
        stream = torch.cuda.current_stream(xd.device).cuda_stream
        rc = self._lib.bddc_spmv(self._ctx, C.c_void_p(xd.data_ptr()), C.c_void_p(y.data_ptr()),
                                 C.c_void_p(stream))
        raise_for(rc, "bddc_spmv failed")
        return y if is_tensor else y.cpu().numpy()

    def harmonic(self, gamma_values):
        torch = self._torch
        gd, is_tensor = self._as_device(gamma_values, "interface values", len(self.gamma_dofs))
        out = torch.empty(self.n, dtype=torch.float64, device=gd.device)
        stream = torch.cuda.current_stream(gd.device).cuda_stream
        rc = self._lib.bddc_harmonic(self._ctx, C.c_void_p(gd.data_ptr()),
                                     C.c_void_p(out.data_ptr()), C.c_void_p(stream))
        raise_for(rc, "bddc_harmonic failed")
        return out if is_tensor else out.cpu().numpy()

    _harmonic = harmonic

    def pcg(self, b, tol=1e-6, max_iters=2000, x_out=None):
        """Fused device PCG (krylov.py:31-92); returns (x, alphas, betas, history, iterations,
        converged). Host numpy b → host x (copies inside); CUDA tensor b → CUDA tensor x."""
        torch = self._torch
        alphas = np.zeros(max_iters + 1)
        betas = np.zeros(max_iters + 1)
        resid = np.zeros(max_iters + 2)
        rep = _capi.PcgReport()
        err = C.create_string_buffer(512)
        if isinstance(b, torch.Tensor) and b.device.type == "cuda":
            bd, _ = self._as_device(b, "right-hand side")
            if x_out is not None:
                x, _ = self._as_device(x_out, "x_out")
            else:
                x = torch.empty_like(bd)
            torch.cuda.current_stream(bd.device).synchronize()
            rc = self._lib.bddc_pcg(self._ctx, C.c_void_p(bd.data_ptr()), C.c_void_p(x.data_ptr()),
                                    float(tol), int(max_iters), _capi.ptr(alphas, C.c_double),
                                    _capi.ptr(betas, C.c_double), _capi.ptr(resid, C.c_double),
                                    C.byref(rep), err, len(err))
        else:
            bh = np.ascontiguousarray(b.cpu().numpy() if isinstance(b, torch.Tensor) else b,
                                      dtype=np.float64)
            if bh.shape != (self.n,):
                raise ValueError(f"right-hand side has shape {bh.shape}, expected ({self.n},)")
            x = np.zeros(self.n)
            rc = self._lib.bddc_pcg_host(self._ctx, _capi.ptr(bh, C.c_double),
                                         _capi.ptr(x, C.c_double), float(tol), int(max_iters),
                                         _capi.ptr(alphas, C.c_double), _capi.ptr(betas, C.c_double),
                                         _capi.ptr(resid, C.c_double), C.byref(rep), err, len(err))
            if rc == 0:
                x = self.allgather_owned(x)
        raise_for(rc, err.value.decode(errors="replace"))
        k = rep.iterations
        return x, alphas[:k].copy(), betas[: max(k - 1, 0)].copy(), resid[: k + 1].copy(), k, bool(rep.converged)

    @property
    def world(self) -> int:
        return self.comm.world if self.comm is not None else 1

    def allgather_owned(self, v: np.ndarray) -> np.ndarray:
        """Sharded: the full vector from every rank's owned rows (host numpy, all ranks)."""
        if self.world == 1:
            return v
        import torch.distributed as dist

        parts = [None] * self.world
        sl = self.slab
        dist.all_gather_object(parts, (sl.fo_lo, np.ascontiguousarray(v[sl.fo_lo:sl.fo_hi])),
                               group=self.comm.group)
        out = np.zeros(self.n)
        for lo, part in parts:
            out[lo:lo + len(part)] = part
        return out

    def debug_buffer(self, name: str) -> np.ndarray:
        """Copy an internal device buffer to host (diagnostics / kernel-level tests)."""
        n = self._lib.bddc_debug_copy(self._ctx, name.encode(), None, 0)
        if n < 0:
            raise KeyError(name)
        out = np.empty(max(n, 0))
        got = self._lib.bddc_debug_copy(self._ctx, name.encode(), _capi.ptr(out, C.c_double), n)
        if got != n:
            raise RuntimeError(f"debug copy of {name} failed")
        return out

    def sync(self):
        self._lib.bddc_sync(self._ctx)

    def kernel_launches_per_apply(self) -> int:
        return int(self._lib.bddc_kernel_launches_per_apply(self._ctx))

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            self._lib.bddc_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_bddc(system: AssembledSystem, pair: PartitionPair, objects: ObjectTable, recipe,
               weights: WeightingOperator, coarse_scaling: str = "reference",
               device: int = 0, comm=None) -> BddcOperator:
    """Assemble the preconditioner on the GPU (bddc.py:393-523).

    The recipe is validated (RecipeError) before any factorization, as in the reference.
    ``comm`` (shard.NcclComm / shard.HostComm): this process is one rank of a sharded
    operator; every rank passes the same global problem.
    """
    if isinstance(recipe, str):
        recipe = Recipe.parse(recipe)
    if coarse_scaling not in COARSE_SCALINGS:
        raise ValueError(f"unknown coarse_scaling {coarse_scaling!r}; expected {COARSE_SCALINGS}")
    if pair.box_layout is None:
        raise ValueError(
            "the device operator needs Θ to be a uniform box partition (partition_uniform); "
            "any refinement Θ̂ (refine_uniform, refine_by_coefficient) is supported on top of it")
    t0 = time.perf_counter()
    constraints = select_constraints(objects, recipe, pair)
    # the slot tables come from the device kernels (index_sets.cu) and the coarse assembly
    # pattern is built by the setup on the device (coarse_pattern.cu);
    host = os.environ.get("BDDC_HOST_PLAN") == "1"  # the numpy / host statements (checkers)
    plan = build_device_plan(pair, constraints, weights, coarse_pattern="host" if host else "device",
                             device=None if host else device)
    prep = time.perf_counter() - t0
    op = BddcOperator(system, pair, weights, recipe, constraints, plan, coarse_scaling, device, comm)
    op.times.prep_s = prep
    op._setup()
    return op


def apply_bddc(bddc: BddcOperator, r):
    """bddc.py:526."""
    return bddc.apply(r)


def harmonic_extension(bddc: BddcOperator, interface_values):
    """Discrete harmonic extension of interface values aligned with gamma_dofs (bddc.py:530-539)."""
    shape = tuple(np.shape(interface_values))
    if shape != (len(bddc.gamma_dofs),):
        raise ValueError(
            f"expected {len(bddc.gamma_dofs)} interface values, got {shape}"
        )
    return bddc.harmonic(interface_values)


__all__ = [
    "BddcOperator", "NotSpdOperatorError", "Recipe", "RecipeError", "apply_bddc", "build_bddc",
    "harmonic_extension", "COARSE_SCALINGS",
]
