"""TEST INFRASTRUCTURE ONLY — generate golden fixtures from the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python oracle/make_golden.py

It imports the unmodified reference package ``bddcso`` from /root/reference/pkg/src and
runs each case through the reference's own public API (build_mesh → partition_uniform →
refine_uniform → assemble → classify_objects → compute_weights → build_bddc → apply → pcg).
Two documented extensions are applied by patching, never by editing reference files:

* P1 cases swap ``bddcso.mesh._element_stiffness_box`` (mesh.py:132, its only element
  hook, used by assemble_cells mesh.py:189) for the P1-Kuhn macro element;
* "spec" coarse-scaling cases replace ``SaddleFactorization.solve`` (linalg.py:158-172) by
  the one-line corrected version that scales g and λ by s instead of 1/s;
* random sources and block coefficients are passed through ``pcg(b=...)`` and the
  ``CoefficientField`` (the reference takes any b and any α, krylov.py:31, mesh.py:52).

Outputs: tests/golden/<case>.npz (index sets, weights, coarse matrix, B·r on seeded r,
PCG iterations / α / β / κ / x). The oracle is then pinned against these files by
tests/test_oracle_golden.py; the GPU path is checked against the oracle.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

import bddcso  # noqa: E402  (reference, read-only)
import bddcso.linalg as rlin  # noqa: E402
import bddcso.mesh as rmesh  # noqa: E402
import bddcso.partition as rpart  # noqa: E402

from oracle import bddc_oracle as orc  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")

_Q1 = rmesh._element_stiffness_box
_SOLVE = rlin.SaddleFactorization.solve
_VALIDATE = rpart.PartitionPair._validate


def _no_validate(self):
    return None


def _p1_box(lengths, alpha):
    return alpha * orc.p1_kuhn_element([float(x) for x in lengths])


def _spec_solve(self, f, g):
    f = np.asarray(f, dtype=float)
    g = np.asarray(g, dtype=float)
    if self.m == 0:
        return self._lu.solve(f), np.zeros((0,) + f.shape[1:])
    s = 1.0 / self._scale  # reference stores 1/s; the corrected solve multiplies by s
    sol = self._lu.solve(np.concatenate([f, s * g], axis=0))
    return sol[: self.n], s * sol[self.n:]


# (name, dim, cells, subs, split, recipe, weighting, element, coeff, rhs, mode, tol, full)
CASES = [
    ("cfg1_p1_ref", 2, (64, 64), (4, 4), 4, "ve", "cardinality", "p1", "const", "one", "reference", 1e-8, False),
    ("cfg1_p1_spec", 2, (64, 64), (4, 4), 4, "ve", "cardinality", "p1", "const", "one", "spec", 1e-8, False),
    ("cfg1_q1_ref", 2, (64, 64), (4, 4), 4, "ve", "cardinality", "q1", "const", "one", "reference", 1e-8, False),
    ("cfg2a_p1_L4h", 2, (128, 128), (4, 4), 8, "ve", "cardinality", "p1", "const", "uniform", "reference", 1e-8, False),
    ("cfg2a_p1_Lh", 2, (64, 64), (2, 2), 32, "ve", "cardinality", "p1", "const", "uniform", "reference", 1e-8, False),
    ("cfg2a_p1_LH", 2, (128, 128), (4, 4), 1, "ve", "counting", "p1", "const", "uniform", "reference", 1e-8, False),
    ("cfg3a_p1_ref", 3, (16, 16, 16), (2, 2, 2), 2, "vef", "cardinality", "p1", "const", "one", "reference", 1e-8, False),
    ("cfg3b_p1_ref", 3, (24, 24, 24), (3, 3, 3), 2, "vef", "cardinality", "p1", "const", "one", "reference", 1e-8, False),
    ("cfg4a_p1_spec", 3, (16, 16, 16), (2, 2, 2), 2, "vef", "coefficient", "p1", "blocks", "one", "spec", 1e-8, False),
    ("cfg4a_p1_ref", 3, (16, 16, 16), (2, 2, 2), 2, "vef", "coefficient", "p1", "blocks", "one", "reference", 1e-8, False),
    ("q1_3d_vf", 3, (12, 12, 12), (3, 3, 3), 2, "vf", "cardinality", "q1", "const", "one", "reference", 1e-8, False),
    ("full_p1_2d", 2, (32, 32), (4, 4), 2, "vef", "cardinality", "p1", "const", "one", "spec", 1e-8, True),
]
# Parity at scale (round 2): the reference run with PartitionPair validation skipped (its
# O(subsubdomains x cells) ndimage loop, partition.py:63-73; SURVEY §8(c) prescribes
# validate=False for uniform box refinements, which are valid by construction). r and b are
# not stored (regenerated from their seeds by tests/conftest.py) to keep the files small.
BIG_CASES = [
    # 3D, cfg3/cfg5 local geometry, 8^3 subdomains: coarse problem 15,967 unknowns,
    # multi-panel coarse fronts (top separator 961)
    ("cfg3c_p1_ref", 3, (64, 64, 64), (8, 8, 8), 2, "vef", "cardinality", "p1", "const", "one", "reference", 1e-8, False),
    # cfg5 local geometry with its random source, 6^3 subdomains
    ("cfg5a_p1_ref", 3, (48, 48, 48), (6, 6, 6), 2, "vef", "cardinality", "p1", "const", "uniform", "reference", 1e-8, False),
    # cfg4 (the coefficient config runs in spec scaling) at 4^3 subdomains
    ("cfg4b_p1_spec", 3, (32, 32, 32), (4, 4, 4), 2, "vef", "coefficient", "p1", "blocks", "one", "spec", 1e-8, False),
    # cfg2 L = h with 4x4 subdomains: corner / edge / interior subdomains have different s_i,
    # so the reference-mode coarse-basis scaling is visible (2x2 subdomains hide it)
    ("cfg2b_p1_Lh44", 2, (128, 128), (4, 4), 32, "ve", "cardinality", "p1", "const", "uniform", "reference", 1e-8, False),
    # cfg2 local geometry (32^2 subdomains, L = 4h) on 16x16 subdomains
    ("cfg2c_p1_L4h", 2, (512, 512), (16, 16), 8, "ve", "cardinality", "p1", "const", "uniform", "reference", 1e-8, False),
]
# Θ̂ from refine_by_coefficient (partition.py:202-220) on a channels field (problems.py:42-102):
# the components of constant α inside each box subdomain (split = -1 marks it)
COEFF_CASES = [
    ("chan_q1_coeff", 3, (16, 16, 16), (2, 2, 2), -1, "vef", "coefficient", "q1", "channels", "one", "reference", 1e-8, False),
    ("chan_p1_coeff2d", 2, (48, 48), (3, 3), -1, "ve", "coefficient", "p1", "channels", "one", "spec", 1e-8, False),
]
CHANNELS = {2: (3.0, 2, 2, 0), 3: (3.0, 2, 2, 1)}  # contrast exponent, cross-section, bars, axis


def _set_element(element):
    rmesh._element_stiffness_box = _p1_box if element == "p1" else _Q1


def _set_mode(mode):
    rlin.SaddleFactorization.solve = _spec_solve if mode == "spec" else _SOLVE


def run_case(case, big=False):
    (name, dim, cells, subs, split, recipe, wmode, element, coeff, rhs, mode, tol, full) = case
    _set_element(element)
    _set_mode(mode)
    rpart.PartitionPair._validate = _no_validate if big else _VALIDATE
    mesh = bddcso.build_mesh(dim, cells)
    if coeff == "const":
        cf = bddcso.make_constant(mesh, 1.0)
    elif coeff == "channels":
        cf = bddcso.make_channels(mesh, subs, bddcso.ChannelSpec(*CHANNELS[dim]))
    else:
        cf = bddcso.CoefficientField(orc.block_alpha(cells, 4, seed=0))
    theta = bddcso.partition_uniform(mesh, subs)
    if split < 0:
        pair = bddcso.refine_by_coefficient(mesh, theta, cf)
    else:
        pair = bddcso.refine_uniform(mesh, theta, split)
    system = bddcso.assemble(mesh, cf, 1.0)
    objects = bddcso.classify_objects(pair)
    weights = bddcso.compute_weights(pair, wmode, cf)
    recipe_obj = bddcso.Recipe.full() if full else recipe
    t0 = time.perf_counter()
    op = bddcso.build_bddc(system, pair, objects, recipe_obj, weights)
    t_build = time.perf_counter() - t0
    n = mesh.free_count
    if rhs == "one":
        b = system.rhs
    else:
        b = orc.load(orc.make_mesh(dim, cells, element), orc.uniform_f(n, seed=0))
    rng = np.random.default_rng(1234)
    r = rng.standard_normal(n)
    Br = op.apply(r)
    A = system.matrix.tocsr()
    t0 = time.perf_counter()
    x, rep = bddcso.pcg(lambda v: A @ v, op.apply, b, tol=tol, max_iters=2000)
    t_pcg = time.perf_counter() - t0

    # index sets
    W = 2**dim
    sig = -np.ones((len(objects), W), dtype=np.int64)
    own = -np.ones((len(objects), W), dtype=np.int64)
    kinds = np.array([("vertex", "edge", "face").index(o.kind) for o in objects], dtype=np.int8)
    dptr = np.zeros(len(objects) + 1, dtype=np.int64)
    dl = []
    for i, o in enumerate(objects):
        sig[i, : len(o.signature)] = o.signature
        own[i, : len(o.owners)] = o.owners
        dptr[i + 1] = dptr[i] + len(o.dofs)
        dl.append(np.asarray(o.dofs))
    dlist = np.concatenate(dl) if dl else np.zeros(0, np.int64)
    cons = op.constraints
    con_obj = np.array([c.object_id for c in cons], dtype=np.int64)
    con_coeff = np.concatenate([c.coeffs for c in cons]) if len(cons) else np.zeros(0)
    con_ptr = np.concatenate([[0], np.cumsum([len(c.dofs) for c in cons])]).astype(np.int64)
    con_dofs = np.concatenate([c.dofs for c in cons]) if len(cons) else np.zeros(0, np.int64)
    # weights per (gamma dof, member)
    wsub, wdof, wval = [], [], []
    for d in pair.membership.gamma_dofs:
        for s in weights.members(int(d)):
            wsub.append(s)
            wdof.append(int(d))
            wval.append(weights.weight(s, int(d)))
    cm = op.coarse_matrix.tocsr() if op.coarse_matrix is not None else None
    out = dict(
        dim=dim, cells=np.array(cells), subs=np.array(subs), split=split, recipe=recipe,
        weighting=wmode, element=element, coeff=coeff, rhs_kind=rhs, mode=mode, tol=tol,
        full=full, n=n, coarse_size=op.coarse_size, gamma_dofs=pair.membership.gamma_dofs,
        obj_sig=sig, obj_owners=own, obj_kind=kinds, obj_dof_ptr=dptr, obj_dofs=dlist,
        con_obj=con_obj, con_ptr=con_ptr, con_dofs=con_dofs, con_coeff=con_coeff,
        w_sub=np.array(wsub), w_dof=np.array(wdof), w_val=np.array(wval),
        b=b, r=r, Br=Br, x=x, iterations=rep.iterations, converged=rep.converged,
        kappa=rep.kappa_estimate, ritz=np.array(rep.ritz_extremes),
        residual_history=np.array(rep.residual_history),
        t_build=t_build, t_pcg=t_pcg,
    )
    if cm is not None and cm.shape[0] <= 4000:
        out.update(coarse_data=cm.data, coarse_indices=cm.indices, coarse_indptr=cm.indptr)
    if split < 0:
        out.update(refine="coefficient", theta_hat=pair.theta_hat, alpha=cf.alpha)
    if big:  # r = default_rng(1234).standard_normal(n); b from the source seed
        out.update(big=True, coarse_diag=cm.diagonal() if cm is not None else np.zeros(0))
        del out["r"], out["b"]
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    names = sys.argv[1:]
    for case, big in [(c, False) for c in CASES + COEFF_CASES] + [(c, True) for c in BIG_CASES]:
        if names and case[0] not in names:
            continue
        if not names and big and os.path.exists(os.path.join(OUT, case[0] + ".npz")):
            continue  # minutes each: regenerate only when named
        t0 = time.perf_counter()
        res = run_case(case, big)
        np.savez_compressed(os.path.join(OUT, case[0] + ".npz"), **res)
        print(f"{case[0]:16s} n={res['n']:7d} coarse={res['coarse_size']:6d} "
              f"its={res['iterations']:4d} kappa={res['kappa']:.10g} "
              f"({time.perf_counter() - t0:.1f}s)")
    # refine_by_coefficient labels (partition.py:202-220) on a channel field
    _set_element("q1")
    mesh = bddcso.build_mesh(3, (12, 12, 12))
    cf = bddcso.make_channels(mesh, (2, 2, 2), bddcso.ChannelSpec(3.0, 2, 2, 1))
    pair = bddcso.refine_by_coefficient(mesh, bddcso.partition_uniform(mesh, (2, 2, 2)), cf)
    np.savez_compressed(os.path.join(OUT, "refine_coeff.npz"), cells=np.array((12, 12, 12)),
                        subs=np.array((2, 2, 2)), alpha=cf.alpha, theta_hat=pair.theta_hat)
    # SPEC KATs for the combinatorial counter
    kat = {f"{s}": bddcso.count_coarse_dofs((10, 10, 10), s, "vef") for s in (1, 2, 4, 6, 8)}
    np.savez(os.path.join(OUT, "count_kat.npz"), **{k: np.array(v) for k, v in kat.items()})
    print("count KAT", kat)
    _set_element("q1")
    _set_mode("reference")
    rpart.PartitionPair._validate = _VALIDATE


if __name__ == "__main__":
    main()
