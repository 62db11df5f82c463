"""TEST INFRASTRUCTURE ONLY — pins of the REFERENCE at the BASELINE configs' full sizes.

Run in the build container (where /root/reference exists; tens of minutes per case):

    python oracle/make_fullsize_pins.py cfg3 [cfg2_L4h ...]

Each case runs the unmodified reference package through its public API exactly as
oracle/make_golden.py does (same patches: P1 element hook, partition validation skipped for
the uniform box refinement, which is valid by construction), at the size BASELINE.json names.
The full vectors (millions of doubles) are not committed; the output
tests/golden/fullsize/<case>.npz holds what a parity test needs: iterations, kappa, the
residual history, norms of x and B r, and x / B r at `NSAMP` seeded sample positions (r and b
are regenerated from their seeds by the tests, as for the scale fixtures).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as mg  # noqa: E402  (imports the reference and sets up the patches)

bddcso, orc = mg.bddcso, mg.orc
OUT = os.path.join(mg.OUT, "fullsize")
NSAMP = 65536

# name -> (dim, cells, subs, split, recipe, weighting, element, coeff, rhs, mode, tol): BASELINE configs
FULL = {
    "cfg3": (3, (128, 128, 128), (16, 16, 16), 2, "vef", "cardinality", "p1", "const", "one", "reference", 1e-8),
    "cfg2_L4h": (2, (2048, 2048), (64, 64), 8, "ve", "cardinality", "p1", "const", "uniform", "reference", 1e-8),
    # cfg4: 1e12 coefficient contrast, coefficient weights; spec scaling as bench.py runs it
    "cfg4": (3, (128, 128, 128), (16, 16, 16), 2, "vef", "coefficient", "p1", "blocks", "one", "spec", 1e-8),
    # half-size cfg3 (fast check of this script)
    "cfg3_half": (3, (64, 64, 64), (8, 8, 8), 2, "vef", "cardinality", "p1", "const", "one", "reference", 1e-8),
}


def run(name):
    dim, cells, subs, split, recipe, wmode, element, coeff, rhs, mode, tol = FULL[name]
    mg._set_element(element)
    mg._set_mode(mode)
    mg.rpart.PartitionPair._validate = mg._no_validate
    t = {}

    def lap(key, t0):
        t[key] = time.perf_counter() - t0
        print(f"  {name}: {key} {t[key]:.1f} s", flush=True)

    t0 = time.perf_counter()
    mesh = bddcso.build_mesh(dim, cells)
    cf = (bddcso.make_constant(mesh, 1.0) if coeff == "const"
          else bddcso.CoefficientField(orc.block_alpha(cells, 4, seed=0)))
    theta = bddcso.partition_uniform(mesh, subs)
    pair = bddcso.refine_uniform(mesh, theta, split)
    lap("mesh_partition", t0)
    t0 = time.perf_counter()
    system = bddcso.assemble(mesh, cf, 1.0)
    lap("assemble", t0)
    t0 = time.perf_counter()
    objects = bddcso.classify_objects(pair)
    weights = bddcso.compute_weights(pair, wmode, cf)
    lap("objects_weights", t0)
    t0 = time.perf_counter()
    op = bddcso.build_bddc(system, pair, objects, recipe, weights)
    lap("build_bddc", t0)
    n = mesh.free_count
    if rhs == "one":
        b = system.rhs
    else:
        b = orc.load(orc.make_mesh(dim, cells, element), orc.uniform_f(n, seed=0))
    r = np.random.default_rng(1234).standard_normal(n)
    t0 = time.perf_counter()
    Br = op.apply(r)
    lap("apply", t0)
    A = system.matrix.tocsr()
    t0 = time.perf_counter()
    x, rep = bddcso.pcg(lambda v: A @ v, op.apply, b, tol=tol, max_iters=2000)
    lap("pcg", t0)
    idx = np.sort(np.random.default_rng(99).choice(n, size=min(NSAMP, n), replace=False))
    cm = op.coarse_matrix.tocsr()
    out = dict(
        dim=dim, cells=np.array(cells), subs=np.array(subs), split=split, recipe=recipe,
        weighting=wmode, element=element, coeff=coeff, rhs_kind=rhs, mode=mode, tol=tol, full=False,
        n=n, coarse_size=op.coarse_size, iterations=rep.iterations, converged=rep.converged,
        kappa=rep.kappa_estimate, ritz=np.array(rep.ritz_extremes),
        residual_history=np.array(rep.residual_history),
        idx=idx, x_s=x[idx], Br_s=Br[idx], x_norm=np.linalg.norm(x), Br_norm=np.linalg.norm(Br),
        x_sum=x.sum(), Br_sum=Br.sum(), coarse_diag_s=cm.diagonal()[:: max(1, op.coarse_size // 4096)],
        coarse_trace=cm.diagonal().sum(), times=np.array([t[k] for k in sorted(t)]),
        time_keys=np.array(sorted(t)),
    )
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print(f"{name}: n={n} coarse={op.coarse_size} its={rep.iterations} kappa={rep.kappa_estimate:.10g} "
          f"total {sum(t.values()):.0f} s", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["cfg3"]:
        run(nm)
