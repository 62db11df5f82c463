"""Two-level vs three-level BDDC-SO on one workload of bench.py (default cfg3), on one GPU.

Diagnostic for DESIGN.md §10a, not the bench contract: prints one JSON line with the PCG
iteration counts and condition estimates of both methods, the time of one direct coarse solve
against one level-2 solve, the level-2 setup time, and the wall time of one re-setup + solve of
both methods (under the hook the 3D re-setup skips the exact coarse factorization).

    python tools/three_level_bench.py [--workload cfg3] [--coarsening 4]
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import torch  # noqa: E402

import bench  # noqa: E402


def lean(a, pb, P):
    """Three-level operator from nothing: cold build, then re-setup + PCG (median of 3)."""
    b = pb["b"]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = P.ThreeLevelOperator.build(pb["system"], pb["pair"], pb["objs"], pb["recipe"], pb["w"],
                                   coarsening=a.coarsening, coarse_scaling=pb["scaling"])
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    steps = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t.refactor()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        x, rep = P.pcg(t.matvec, t.apply, b, tol=1e-8, max_iters=500)
        torch.cuda.synchronize()
        steps.append(((t1 - t0) * 1e3, (time.perf_counter() - t1) * 1e3))
    steps = sorted(steps[1:], key=lambda v: v[0] + v[1])
    rs, ps = steps[len(steps) // 2]
    r = b - t.matvec(x)
    import numpy as np

    free, total = torch.cuda.mem_get_info()
    print(json.dumps({
        "workload": a.workload, "mode": "three-level, set up under the hook", "dofs": int(t.n),
        "n_coarse": int(t.level2.n0), "coarsening": a.coarsening,
        "level2": {"boxes": t.level2.shape[0], "n_coarse2": t.level2.n_coarse2, "n_gamma2": t.level2.n_gamma2},
        "iterations": rep.iterations, "kappa": rep.kappa_estimate, "converged": bool(rep.converged),
        "true_residual_rel": float(np.linalg.norm(r) / np.linalg.norm(b)),
        "cold_build_s": round(build_s, 2), "refactor_ms": round(rs, 2), "pcg_ms": round(ps, 2),
        "step_ms": round(rs + ps, 2), "Mdof_s": round(t.n / (rs + ps) / 1e3, 3),
        "gpu_memory_used_gb": round((total - free) / 2**30, 1)}))
    t.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--coarsening", type=int, default=4)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--cells", type=int, default=0, help="custom 3D workload: cells per axis (cfg5's recipe)")
    ap.add_argument("--subs", type=int, default=0, help="custom 3D workload: subdomains per axis")
    ap.add_argument("--lean", action="store_true",
                    help="only the three-level operator, set up under the hook (no coarse plan / fronts / factor)")
    a = ap.parse_args()
    if a.cells and a.subs:  # cfg5's geometry and recipe at another size
        a.workload = f"cfg5_{a.cells}_{a.subs}"
        bench.WORKLOADS[a.workload] = (3, (a.cells,) * 3, (a.subs,) * 3, 2, "vef", "cardinality", "uniform", "one",
                                       "reference")
    pb = bench.build_host_problem(a.workload, device=0)
    P = pb["P"]
    if a.lean:
        return lean(a, pb, P)
    op = P.build_bddc(pb["system"], pb["pair"], pb["objs"], pb["recipe"], pb["w"],
                      coarse_scaling=pb["scaling"])
    b = pb["b"]

    def timed_pcg(o):
        P.pcg(o.matvec, o.apply, b, tol=1e-8, max_iters=500)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = P.pcg(o.matvec, o.apply, b, tol=1e-8, max_iters=500)
        torch.cuda.synchronize()
        return x, rep, (time.perf_counter() - t0) * 1e3

    x2, rep2, ms2 = timed_pcg(op)
    n0 = op.plan.coarse.n
    r0 = torch.randn(n0, dtype=torch.float64, device="cuda")
    s0 = torch.empty_like(r0)
    stream = torch.cuda.current_stream().cuda_stream

    def ev_ms(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    direct_ms = ev_ms(lambda: op._lib.bddc_coarse_solve(op._ctx, C.c_void_p(r0.data_ptr()),
                                                       C.c_void_p(s0.data_ptr()), C.c_void_p(stream)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = P.ThreeLevelOperator(op, coarsening=a.coarsening)
    torch.cuda.synchronize()
    setup2_s = time.perf_counter() - t0
    level2_ms = ev_ms(lambda: t.level2.solve(r0))
    mats = t._element_matrices()
    numeric_ms = ev_ms(lambda: t.level2.refactor(mats))
    x3, rep3, ms3 = timed_pcg(t)

    def wall_ms(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3 / reps

    refactor3_ms = wall_ms(t.refactor)      # local setup + level-2 numeric (exact coarse factor skipped in 3D)
    l1_hook_ms = wall_ms(t.op.refactor)     # level-1 re-setup alone under the hook
    st3 = op.stats()
    l2_wall_ms = wall_ms(lambda: t.level2.refactor(t._element_matrices()))
    x3b, rep3b, ms3b = timed_pcg(t)
    t.restore()
    refactor2_ms = wall_ms(op.refactor)     # local setup + exact coarse factorization
    import numpy as np

    out = {
        "workload": bench.describe(a.workload) if a.workload in ("cfg3", "cfg4", "cfg5") else a.workload,
        "dofs": int(op.n), "n_coarse": int(n0), "coarsening": a.coarsening,
        "level2": {"boxes": t.level2.shape[0], "n_interior_max": t.level2.shape[1],
                   "n_gamma2_max": t.level2.shape[2], "constraints_max": t.level2.shape[3],
                   "n_gamma2": t.level2.n_gamma2, "n_coarse2": t.level2.n_coarse2},
        "two_level": {"iterations": rep2.iterations, "kappa": rep2.kappa_estimate, "pcg_ms": round(ms2, 2),
                      "coarse_solve_ms": round(direct_ms, 3)},
        "three_level": {"iterations": rep3.iterations, "kappa": rep3.kappa_estimate, "pcg_ms": round(ms3, 2),
                        "level2_solve_ms": round(level2_ms, 3), "level2_setup_s": round(setup2_s, 3),
                        "level2_numeric_ms": round(numeric_ms, 2)},
        "step_ms": {"two_level_refactor": round(refactor2_ms, 2), "two_level_pcg": round(ms2, 2),
                    "three_level_refactor": round(refactor3_ms, 2),
                    "three_level_refactor_level1": round(l1_hook_ms, 2), "three_level_refactor_level2": round(l2_wall_ms, 2),
                    "level1_under_hook_local_ms": round(st3.t_local_ms, 2),
                    "level1_under_hook_coarse_ms": round(st3.t_coarse_ms, 2), "three_level_pcg": round(ms3b, 2),
                    "three_level_its_after_refactor": rep3b.iterations},
        "x_rel_diff": float(np.linalg.norm(x3 - x2) / np.linalg.norm(x2)),
        "coarse_factorization_ms_it_replaces": round(op.stats().t_coarse_ms, 2),
    }
    print(json.dumps(out))
    op.close()


if __name__ == "__main__":
    main()
