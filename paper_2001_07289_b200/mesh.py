"""Structured unit-box meshes, element matrices (Q1 and P1-Kuhn) and host assembly.

Mirrors ``bddcso.mesh`` (reference ``pkg/src/bddcso/mesh.py``):

* ``build_mesh``            ↔ mesh.py:73-129  (x-fastest node ids, Dirichlet on the whole boundary)
* ``element_stiffness``     ↔ mesh.py:163-169 (Q1, 2-point Gauss) + ``element="p1"``
* ``assemble_cells``        ↔ mesh.py:172-198 (cell-subset assembly, symmetric Dirichlet elimination)
* ``assemble``              ↔ mesh.py:201-222 (global matrix over free dofs + load f·h^d per node)

The device path never builds the global CSR: it applies the operator matrix-free from
the per-cell coefficient and the 2^d×2^d reference element matrix (see ``csrc/stencil.cuh``).
The host CSR here exists for API compatibility and small-case checks; it is built lazily.

P1 element. The reference implements Q1 only. BASELINE configs use P1
simplices on the Kuhn split of each box (2 triangles / 6 tetrahedra along the main
diagonal corner 0 → corner 2^d−1). Its macro-element matrix is the sum of the simplex
stiffnesses; it is computed in closed form (barycentric gradients are ±e_k/h_k), so
the same bits come out on every platform.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field
from functools import cached_property
from typing import Sequence

import numpy as np

from .linalg import SparseSym

ELEMENTS = ("q1", "p1")
_SQRT3 = math.sqrt(3.0)


@dataclass(frozen=True)
class StructuredMesh:
    """Tensor-product grid of the unit box (mesh.py:20-49).

    ``cell_nodes`` (corner c has bit d <-> +1 on axis d), ``node_coords`` and
    ``boundary_mask`` are the reference's fields; they are built on first access (the device
    path never needs them; at cfg5 they are 1.2 GB of int64)."""

    dim: int
    cells_per_dim: tuple
    node_count: int
    cell_count: int
    spacings: tuple
    free_nodes: np.ndarray
    node_to_free: np.ndarray
    element: str = "q1"

    @property
    def free_count(self) -> int:
        return len(self.free_nodes)

    @property
    def nodes_per_dim(self) -> tuple:
        return tuple(c + 1 for c in self.cells_per_dim)

    def _grid(self, sizes):
        """(prod(sizes), dim) x-fastest multi-indices."""
        axes = np.meshgrid(*[np.arange(n, dtype=np.int64) for n in reversed(sizes)], indexing="ij")
        return np.stack([a.ravel() for a in reversed(axes)], axis=1)

    @cached_property
    def node_coords(self) -> np.ndarray:
        return self._grid(self.nodes_per_dim) * np.asarray(self.spacings)

    @cached_property
    def boundary_mask(self) -> np.ndarray:
        mask = np.ones(self.node_count, dtype=bool)
        mask[self.free_nodes] = False
        return mask

    @cached_property
    def cell_nodes(self) -> np.ndarray:
        npd = self.nodes_per_dim
        strides = np.cumprod((1,) + npd[:-1]).astype(np.int64)
        base = _axis_sum([np.arange(c, dtype=np.int64) * strides[d] for d, c in enumerate(self.cells_per_dim)])
        corners = np.array([sum(((c >> d) & 1) * int(strides[d]) for d in range(self.dim))
                            for c in range(2**self.dim)], dtype=np.int64)
        return base[:, None] + corners[None, :]

    @cached_property
    def _cell_multi(self) -> np.ndarray:
        return self._grid(self.cells_per_dim)

    def cell_multi_indices(self) -> np.ndarray:
        return self._cell_multi

    def cells_grid(self, values: np.ndarray) -> np.ndarray:
        return np.asarray(values).reshape(tuple(reversed(self.cells_per_dim)))


def _axis_sum(parts) -> np.ndarray:
    """x-fastest flattened outer sum: out[i0 + n0*(i1 + n1*i2)] = parts[0][i0] + parts[1][i1] + ..."""
    out = parts[-1]
    for p in reversed(parts[:-1]):
        out = (out[:, None] + p[None, :]).ravel()
    return out


@dataclass(frozen=True)
class CoefficientField:
    """Piecewise-constant diffusion coefficient, one positive value per cell (mesh.py:52-61)."""

    alpha: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "alpha", np.asarray(self.alpha, dtype=float))
        if np.any(self.alpha <= 0.0):
            raise ValueError("diffusion coefficient must be positive on every cell")


class AssembledSystem:
    """Global system over free dofs (mesh.py:64-70).

    ``matrix`` (a :class:`SparseSym`) is assembled on first access; the device path
    only needs ``mesh``, ``coeff`` and ``rhs``.
    """

    def __init__(self, mesh: StructuredMesh, coeff: CoefficientField, rhs: np.ndarray,
                 matrix: SparseSym | None = None):
        self.mesh = mesh
        self.coeff = coeff
        self.rhs = rhs
        self.free_dof_map = mesh.free_nodes
        self._matrix = matrix

    @property
    def matrix(self) -> SparseSym:
        if self._matrix is None:
            self._matrix = assemble_cells(
                self.mesh, self.coeff, np.arange(self.mesh.cell_count), self.mesh.free_nodes
            )
        return self._matrix

    @property
    def n(self) -> int:
        return self.mesh.free_count


def build_mesh(dim: int, cells_per_dim: Sequence[int], element: str = "q1") -> StructuredMesh:
    """Structured mesh of the unit box (mesh.py:73-129); ``element`` selects Q1 or P1-Kuhn."""
    if dim not in (2, 3):
        raise ValueError(f"dim must be 2 or 3, got {dim}")
    if element not in ELEMENTS:
        raise ValueError(f"unknown element {element!r}; expected one of {ELEMENTS}")
    cells = tuple(int(c) for c in cells_per_dim)
    if len(cells) != dim:
        raise ValueError(f"expected {dim} cell counts, got {len(cells)}")
    if any(c < 1 for c in cells):
        raise ValueError(f"cells_per_dim must be positive, got {cells}")

    npd = tuple(c + 1 for c in cells)
    node_count = int(np.prod(npd))
    cell_count = int(np.prod(cells))
    spacings = tuple(1.0 / c for c in cells)
    # free nodes: interior grid points in increasing node id (mesh.py:97-102), as an outer sum
    strides = np.cumprod((1,) + npd[:-1]).astype(np.int64)
    free_nodes = _axis_sum([np.arange(1, c, dtype=np.int64) * strides[d] for d, c in enumerate(cells)])
    node_to_free = np.full(node_count, -1, dtype=np.int64)
    node_to_free[free_nodes] = np.arange(len(free_nodes))
    return StructuredMesh(dim, cells, node_count, cell_count, spacings, free_nodes, node_to_free, element)


def q1_element_box(lengths: Sequence[float]) -> np.ndarray:
    """Q1 Laplacian on a box, tensor 2-point Gauss rule (same rule as mesh.py:132-160)."""
    lengths = [float(x) for x in lengths]
    dim = len(lengths)
    m = 2**dim
    pts = (0.5 - 0.5 / _SQRT3, 0.5 + 0.5 / _SQRT3)
    vol = float(np.prod(lengths))
    K = np.zeros((m, m))
    for q in range(m):
        xi = [pts[(q >> d) & 1] for d in range(dim)]
        G = np.empty((m, dim))
        for c in range(m):
            for d in range(dim):
                g = 1.0
                for e in range(dim):
                    bit = (c >> e) & 1
                    if e == d:
                        g *= 1.0 if bit else -1.0
                    else:
                        g *= xi[e] if bit else 1.0 - xi[e]
                G[c, d] = g / lengths[d]
        K += (vol / m) * (G @ G.T)
    return 0.5 * (K + K.T)


def p1_kuhn_element_box(lengths: Sequence[float]) -> np.ndarray:
    """P1 Laplacian macro-element of the Kuhn split of a box (sum over d! simplices).

    Simplex for axis permutation π: 1 ≥ t_π0 ≥ … ≥ t_π(d-1) ≥ 0 with t_k = x_k/h_k; its
    vertices are corners 0, e_π0, e_π0+e_π1, …, and the barycentric gradients are
    −e_π0/h_π0, (e_π(k-1)/h_π(k-1) − e_πk/h_πk), e_π(d-1)/h_π(d-1). Entries are
    vol·Σ_axis g_i g_j, accumulated in a fixed order.
    """
    h = [float(x) for x in lengths]
    dim = len(h)
    m = 2**dim
    vol = float(np.prod(h)) / math.factorial(dim)
    inv2 = [1.0 / (hk * hk) for hk in h]
    K = np.zeros((m, m))
    for perm in itertools.permutations(range(dim)):
        corners = [0]
        for k in range(dim):
            corners.append(corners[-1] | (1 << perm[k]))
        # sign of each barycentric gradient component: grads[v][axis] in {-1,0,1} (times 1/h_axis)
        grads = [[0] * dim for _ in range(dim + 1)]
        grads[0][perm[0]] = -1
        for k in range(1, dim):
            grads[k][perm[k - 1]] = 1
            grads[k][perm[k]] = -1
        grads[dim][perm[dim - 1]] = 1
        for a in range(dim + 1):
            for b in range(dim + 1):
                s = 0.0
                for ax in range(dim):
                    p = grads[a][ax] * grads[b][ax]
                    if p:
                        s += p * inv2[ax]
                K[corners[a], corners[b]] += vol * s
    return K


def element_matrix_box(lengths: Sequence[float], element: str = "q1") -> np.ndarray:
    if element == "q1":
        return q1_element_box(lengths)
    if element == "p1":
        return p1_kuhn_element_box(lengths)
    raise ValueError(f"unknown element {element!r}")


def element_stiffness(dim: int, h: float, alpha: float, element: str = "q1") -> np.ndarray:
    """Element matrix of a cubic cell of edge h (mesh.py:163-169)."""
    if h <= 0.0:
        raise ValueError("cell edge length must be positive")
    if alpha <= 0.0:
        raise ValueError("coefficient must be positive")
    return alpha * element_matrix_box((h,) * dim, element)


def assemble_cells(mesh: StructuredMesh, coeff: CoefficientField, cells: np.ndarray,
                   keep_nodes: np.ndarray) -> SparseSym:
    """Assemble the given cells restricted to ``keep_nodes`` (mesh.py:172-198)."""
    cells = np.asarray(cells)
    keep_nodes = np.asarray(keep_nodes)
    lookup = np.full(mesh.node_count, -1, dtype=np.int64)
    lookup[keep_nodes] = np.arange(len(keep_nodes))
    K = element_matrix_box(mesh.spacings, mesh.element)
    conn = lookup[mesh.cell_nodes[cells]]
    nc, m = conn.shape
    ii, jj = np.nonzero(np.triu(np.ones((m, m), dtype=bool)) & (K != 0.0) | np.eye(m, dtype=bool))
    rows = conn[:, ii]
    cols = conn[:, jj]
    data = coeff.alpha[cells][:, None] * K[ii, jj][None, :]
    # upper triangle in the local numbering: swap where the local order is reversed
    lo = np.minimum(rows, cols)
    hi = np.maximum(rows, cols)
    mask = lo >= 0
    return SparseSym.from_upper_triplets(len(keep_nodes), lo[mask], hi[mask], data[mask])


def load_vector(mesh: StructuredMesh, f) -> np.ndarray:
    """Consistent load over free dofs: f·vol/2^d per adjacent cell (mesh.py:213-217).

    ``f`` may be a scalar (the reference's only case) or a per-free-dof array, in which
    case b = h^d·f is used (the harness convention of SURVEY §0.3: with f≡1 this equals
    the reference load at every free node).
    """
    vol = float(np.prod(mesh.spacings))
    if np.ndim(f) == 0:
        # every free node lies in exactly 2^d cells: the same value as the reference's sum
        # f·vol/2^d · count (count = 2^d), without the cell -> node incidence
        return np.full(mesh.free_count, float(f) * vol / (2**mesh.dim) * (2**mesh.dim))
    f = np.asarray(f, dtype=float)
    if f.shape != (mesh.free_count,):
        raise ValueError(f"per-dof source has shape {f.shape}, expected ({mesh.free_count},)")
    return vol * f


def assemble(mesh: StructuredMesh, coeff: CoefficientField, f=1.0,
             build_matrix: bool = False) -> AssembledSystem:
    """Global Dirichlet-eliminated system (mesh.py:201-222); the CSR is built lazily."""
    if len(coeff.alpha) != mesh.cell_count:
        raise ValueError(f"coefficient has {len(coeff.alpha)} values for {mesh.cell_count} cells")
    system = AssembledSystem(mesh, coeff, load_vector(mesh, f))
    if build_matrix:
        system.matrix  # noqa: B018 - force assembly
    return system
