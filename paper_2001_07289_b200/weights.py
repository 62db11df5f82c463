"""Recipes, interface weights and constraint selection (host index sets, bit-exact).

Restates the host half of ``bddcso.bddc`` (reference ``pkg/src/bddcso/bddc.py``):

* ``Recipe`` / ``RecipeError``           ↔ bddc.py:36-70
* ``WeightingOperator``                   ↔ bddc.py:73-105
* ``compute_weights``                     ↔ bddc.py:108-145 (+ ``_constant_per_subsubdomain`` 148-162)
* ``Constraint`` / ``select_constraints`` ↔ bddc.py:165-220
* ``_check_sufficiency``                  ↔ bddc.py:239-277 (union-find acceptable paths)

Weights are per object, not per dof: every Γ dof of an object shares its Θ̂-signature,
hence its Θ-membership (= the object's owners) and its weights. Counting and cardinality
weights are ratios of small integers (IEEE division of exact integers is the correctly
rounded rational, so bit-exact with ``float(Fraction)``); coefficient weights are computed
as exact ``Fraction`` sums per object and rounded once, exactly as bddc.py:137-142.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

from .partition import KINDS, ObjectTable, PartitionPair, _KIND_CODE

WEIGHT_MODES = ("cardinality", "counting", "coefficient")


class RecipeError(ValueError):
    """A constraint recipe failed the sufficiency checks (bddc.py:36)."""


@dataclass(frozen=True)
class Recipe:
    """Which object kinds receive a coarse constraint (bddc.py:40-70)."""

    vertices: bool = False
    edges: bool = False
    faces: bool = False
    full_continuity: bool = False

    @classmethod
    def parse(cls, text: str) -> "Recipe":
        letters = set(text)
        if not letters <= {"v", "e", "f"}:
            raise ValueError(f"unknown recipe {text!r}; use letters from 'vef'")
        return cls(vertices="v" in letters, edges="e" in letters, faces="f" in letters)

    @classmethod
    def full(cls) -> "Recipe":
        return cls(vertices=True, edges=True, faces=True, full_continuity=True)

    def selects(self, kind: str) -> bool:
        if self.full_continuity:
            return True
        return {"vertex": self.vertices, "edge": self.edges, "face": self.faces}[kind]

    def kind_mask(self) -> np.ndarray:
        return np.array([self.selects(k) for k in KINDS], dtype=bool)

    def __str__(self):
        if self.full_continuity:
            return "full"
        return "".join(
            c for c, on in zip("vef", (self.vertices, self.edges, self.faces)) if on
        ) or "none"


class WeightingOperator:
    """Interface averaging weights δ†_i(ξ), one per (subdomain, Γ dof) (bddc.py:73-105).

    Stored per object: ``obj_owners`` (n_obj, W) and aligned ``obj_weights`` (float64,
    correctly rounded). ``members(dof)`` is the dof's Θ-membership tuple.
    """

    def __init__(self, mode: str, gamma_dofs: np.ndarray, objects: ObjectTable,
                 obj_weights: np.ndarray, obj_fractions=None, obj_counts=None):
        self.mode = mode
        self.gamma_dofs = gamma_dofs
        self._objects = objects
        self.obj_weights = obj_weights
        self._obj_fractions = obj_fractions  # exact values (coefficient mode)
        self._obj_counts = obj_counts  # numerators over sig_len (cardinality mode)

    @property
    def objects(self) -> ObjectTable:
        return self._objects

    def _slot(self, sub: int, dof: int):
        o = int(self._objects.dof_obj[dof]) if 0 <= dof < len(self._objects.dof_obj) else -1
        if o < 0:
            raise KeyError(f"subdomain {sub} does not contain dof {dof}")
        n = int(self._objects.owner_len[o])
        owners = self._objects.owners[o, :n]
        k = np.flatnonzero(owners == sub)
        if k.size == 0:
            raise KeyError(f"subdomain {sub} does not contain dof {dof}")
        return o, int(k[0])

    def members(self, dof: int) -> tuple:
        o = int(self._objects.dof_obj[dof])
        return tuple(int(v) for v in self._objects.owners[o, : self._objects.owner_len[o]])

    def weight(self, sub: int, dof: int) -> float:
        o, k = self._slot(sub, dof)
        return float(self.obj_weights[o, k])

    def weight_fraction(self, sub: int, dof: int) -> Fraction:
        o, k = self._slot(sub, dof)
        if self.mode == "coefficient":
            return self._obj_fractions[o][k]
        if self.mode == "cardinality":
            return Fraction(int(self._obj_counts[o, k]), int(self._objects.sig_len[o]))
        return Fraction(1, int(self._objects.owner_len[o]))

    def weight_array(self, sub: int, dofs) -> np.ndarray:
        return np.array([self.weight(sub, int(d)) for d in dofs])

    def weights_for(self, sub: np.ndarray, dof: np.ndarray) -> np.ndarray:
        """Vectorised weight lookup for (sub, dof) pairs (0 where sub does not own dof)."""
        obj = self._objects.dof_obj[dof]
        own = self._objects.owners[obj]
        hit = own == sub[:, None]
        w = np.where(hit, self.obj_weights[obj], 0.0).sum(axis=1)
        return w


def _constant_per_subsubdomain(pair: PartitionPair, coeff) -> np.ndarray:
    """α per subsubdomain; error if not constant on one (bddc.py:148-162)."""
    hats = pair.theta_hat
    alpha = np.asarray(coeff.alpha, dtype=float)
    first = np.full(pair.subsubdomain_count, len(hats), dtype=np.int64)
    np.minimum.at(first, hats, np.arange(len(hats)))
    rep = alpha[first[hats]]
    bad = np.flatnonzero(alpha != rep)
    if bad.size:
        # reference reports the smallest offending subsubdomain id (sorted by hat)
        h = int(np.min(hats[bad]))
        raise ValueError(
            f"coefficient-scaled weighting requires a constant coefficient per "
            f"subsubdomain; subsubdomain {h} is not constant"
        )
    return alpha[first]


def compute_weights(pair: PartitionPair, mode: str, coeff=None,
                    objects: ObjectTable | None = None) -> WeightingOperator:
    """Cardinality (Eq. 3), counting, or coefficient (Remark 1) weights (bddc.py:108-145)."""
    if mode not in WEIGHT_MODES:
        raise ValueError(f"unknown weighting mode {mode!r}; expected one of {WEIGHT_MODES}")
    from .partition import classify_objects

    ms = pair.membership
    alpha_hat = None
    if mode == "coefficient":
        if coeff is None:
            raise ValueError("coefficient-scaled weighting requires a coefficient field")
        alpha_hat = _constant_per_subsubdomain(pair, coeff)
    if objects is None:
        objects = classify_objects(pair)
    dev = getattr(objects, "_device_weights", None)
    if dev is not None and mode in dev:  # computed with the objects (index_device.py)
        weights, counts = dev[mode]
        return WeightingOperator(mode, ms.gamma_dofs, objects, weights, None, counts)
    W = objects.owners.shape[1]
    n_obj = len(objects)
    weights = np.zeros((n_obj, W))
    fractions = None
    counts = None
    valid_owner = objects.owners >= 0
    if mode == "counting":
        weights = np.where(valid_owner, 1.0 / np.maximum(objects.owner_len, 1)[:, None], 0.0)
    else:
        sig = objects.signature
        sig_parent = np.where(sig >= 0, pair.parent[np.maximum(sig, 0)], -2)
        if mode == "cardinality":
            # contrib[o, k] = #hats of the signature whose parent is owners[o, k]
            counts = (sig_parent[:, None, :] == objects.owners[:, :, None]).sum(axis=2)
            weights = np.where(valid_owner,
                               counts / np.maximum(objects.sig_len, 1)[:, None], 0.0)
        else:
            fractions = []
            ah = np.where(sig >= 0, alpha_hat[np.maximum(sig, 0)], 0.0)
            for o in range(n_obj):
                n_own = int(objects.owner_len[o])
                contrib = [Fraction(0)] * n_own
                own = objects.owners[o, :n_own].tolist()
                for h in range(int(objects.sig_len[o])):
                    contrib[own.index(int(sig_parent[o, h]))] += Fraction(float(ah[o, h]))
                den = sum(contrib)
                fr = tuple(c / den for c in contrib)
                fractions.append(fr)
                weights[o, :n_own] = [float(f) for f in fr]
    return WeightingOperator(mode, ms.gamma_dofs, objects, weights, fractions, counts)


# --------------------------------------------------------------------------------------
# constraints
# --------------------------------------------------------------------------------------

@dataclass(frozen=True)
class Constraint:
    """bddc.py:165-172."""

    coarse_id: int
    object_id: int
    kind: str
    dofs: np.ndarray
    coeffs: np.ndarray
    owners: tuple


class ConstraintTable:
    """Array form of the selected constraints; indexes like the reference's list.

    con_obj (n_c,)       object id of each constraint (coarse_id = position)
    con_kind (n_c,)      kind code
    dof_ptr / dof_list   CSR of constraint dofs; coeff per entry
    """

    def __init__(self, objects: ObjectTable, con_obj, con_kind, dof_ptr, dof_list, coeff):
        self.objects = objects
        self.con_obj = con_obj
        self.con_kind = con_kind
        self.dof_ptr = dof_ptr
        self.dof_list = dof_list
        self.coeff = coeff

    def __len__(self):
        return len(self.con_obj)

    def owners_of(self, c: int) -> tuple:
        o = int(self.con_obj[c])
        return tuple(int(v) for v in self.objects.owners[o, : self.objects.owner_len[o]])

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        i = int(i)
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        a, b = self.dof_ptr[i], self.dof_ptr[i + 1]
        return Constraint(i, int(self.con_obj[i]), KINDS[int(self.con_kind[i])],
                          self.dof_list[a:b].copy(), self.coeff[a:b].copy(), self.owners_of(i))

    def __iter__(self):
        for i in range(len(self)):
            yield self[i]


def select_constraints(objects: ObjectTable, recipe, pair: PartitionPair) -> ConstraintTable:
    """One row per selected object: vertex value / edge-face mean (bddc.py:175-220)."""
    if isinstance(recipe, str):
        recipe = Recipe.parse(recipe)
    sel = recipe.kind_mask()[objects.kind.astype(np.int64)] if len(objects) else np.zeros(0, bool)
    sel_obj = np.flatnonzero(sel)
    counts = objects.dof_count()
    if recipe.full_continuity:
        # one point constraint per dof of every object, objects in order
        n_per = counts[sel_obj]
        con_obj = np.repeat(sel_obj, n_per)
        con_kind = np.full(len(con_obj), _KIND_CODE["vertex"], dtype=np.int8)
        dof_list = np.concatenate([objects.dof_list[objects.dof_ptr[o]:objects.dof_ptr[o + 1]]
                                   for o in sel_obj]) if len(sel_obj) else np.zeros(0, np.int64)
        dof_ptr = np.arange(len(con_obj) + 1, dtype=np.int64)
        coeff = np.ones(len(con_obj))
    else:
        con_obj = sel_obj
        con_kind = objects.kind[sel_obj]
        n_per = counts[sel_obj]
        dof_ptr = np.concatenate([[0], np.cumsum(n_per)]).astype(np.int64)
        idx = (np.repeat(objects.dof_ptr[sel_obj] - dof_ptr[:-1], n_per)
               + np.arange(dof_ptr[-1]))
        dof_list = objects.dof_list[idx]
        per_con = np.where(con_kind == _KIND_CODE["vertex"], 1.0, 1.0 / np.maximum(n_per, 1))
        coeff = np.repeat(per_con, n_per)
    table = ConstraintTable(objects, con_obj.astype(np.int64), con_kind, dof_ptr,
                            dof_list.astype(np.int64), coeff)
    _check_sufficiency(objects, table, recipe, pair)
    return table


class _UnionFind:
    """Same union/find semantics as bddc.py:223-236 (used to phrase the error message)."""

    def __init__(self, n):
        self.parent = list(range(n))

    def find(self, a):
        while self.parent[a] != a:
            self.parent[a] = self.parent[self.parent[a]]
            a = self.parent[a]
        return a

    def union(self, a, b):
        ra, rb = self.find(a), self.find(b)
        if ra != rb:
            self.parent[rb] = ra


def _check_sufficiency(objects: ObjectTable, cons: ConstraintTable, recipe, pair):
    """Floating-subdomain and acceptable-path checks (bddc.py:239-277)."""
    grounded = pair.grounded_subdomains
    constrained = np.zeros(pair.subdomain_count, dtype=bool)
    if len(cons):
        own = objects.owners[np.unique(cons.con_obj)]
        constrained[own[own >= 0]] = True
    floating = np.flatnonzero(~grounded & ~constrained)
    if floating.size:
        raise RecipeError(
            f"recipe {recipe} leaves floating subdomain {int(floating[0])} without "
            f"any constraint (local Neumann problem singular)"
        )
    if recipe.full_continuity or len(objects) == 0:
        return
    n_hat = pair.subsubdomain_count
    # hats of one subdomain are linked; hats of every selected object's signature are linked
    first_hat = np.full(pair.subdomain_count, n_hat, dtype=np.int64)
    np.minimum.at(first_hat, pair.parent, np.arange(n_hat))
    rows = [np.arange(n_hat)]
    cols = [first_hat[pair.parent]]
    sel_obj = np.unique(cons.con_obj)
    sig = objects.signature[sel_obj]
    valid = sig >= 0
    rows.append(np.broadcast_to(sig[:, :1], sig.shape)[valid])
    cols.append(sig[valid])
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    g = sp.coo_matrix((np.ones(len(r), np.int8), (r, c)), shape=(n_hat, n_hat))
    _, comp = connected_components(g, directed=False)
    all_sig = objects.signature
    lab = np.where(all_sig >= 0, comp[np.maximum(all_sig, 0)], -1)
    bad = np.any((lab != lab[:, :1]) & (all_sig >= 0), axis=1)
    if not bad.any():
        return
    # error path: replay the reference's union order to name the same subsubdomains
    uf = _UnionFind(n_hat)
    by_parent = {}
    for hat, parent in enumerate(pair.parent):
        by_parent.setdefault(int(parent), []).append(hat)
    for hats in by_parent.values():
        for h in hats[1:]:
            uf.union(hats[0], h)
    for o in sel_obj:
        s = [int(v) for v in objects.signature[o, : objects.sig_len[o]]]
        for h in s[1:]:
            uf.union(s[0], h)
    for o in range(len(objects)):
        s = [int(v) for v in objects.signature[o, : objects.sig_len[o]]]
        if len({uf.find(h) for h in s}) > 1:
            s = sorted(s, key=uf.find)
            a, b = s[0], s[-1]
            raise RecipeError(
                f"recipe {recipe} provides no acceptable path between "
                f"subsubdomains {a} (subdomain {int(pair.parent[a])}) and "
                f"{b} (subdomain {int(pair.parent[b])})"
            )
