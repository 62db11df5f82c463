#!/usr/bin/env python
"""BDDC-SO setup + PCG solve throughput on B200 (BASELINE.json metric: Mdof/s, applies/s,
fraction of roofline).

Default workload = the largest BASELINE config that fits one GPU: configs[4] (cfg5), 3D
Poisson on 256^3 cells split into P1 tetrahedra (16,581,375 dofs), 32^3 subdomains of 8^3
cells, subfaces / subedges of 4h + the vertices between them ('vef'), cardinality weights,
f ~ U[-1,1] per dof (seed 0), PCG rtol 1e-8 from x0 = 0, FP64, reference coarse scaling.
The other configs run with --workload (cfg1, cfg2_{LH,L16h,L4h,Lh}, cfg3, cfg4).

One step = numeric BDDC-SO setup on device-resident inputs (local factorizations, coarse
basis, coarse assembly + multifrontal factorization) + the PCG solve to rtol 1e-8.
`value` = dofs solved per second over the timed steps (CUDA events on the library stream);
`e2e` = the same through the C ABI with host buffers (bddc_solve_host: alpha and b uploaded
from pinned memory, overlapped with the setup; x downloaded) every step; `cold_e2e` = one
solve from nothing (host index sets, build_bddc, pcg) through the Python API. Inputs (cfg5:
factors 54 GB + fronts 75 GB) exceed the 126 MB L2 between steps.

`cpu_baseline` and --impl reference run ONE routine (cpu_measure): the reference algorithm
(oracle/bddc_oracle.py, pinned to the reference by tests/golden: SuperLU factorizations,
three-step apply) on bounded samples of the workload's local geometry, one process per host
core with single-threaded BLAS, all processes timed together.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0
FP64_PEAK_TFLOPS = 35.43  # cuBLAS (torch.matmul) FP64 8192^3 measured on this pool, profiles/r01_fp64_peak_probe.log
FP64_DMMA_ISSUE_TFLOPS = 37.07  # mma.sync m8n8k4 issue-bound loop, same probe

WORKLOADS = {
    # name: (dim, cells, subs, split, recipe, weighting, source, coefficient, coarse scaling)
    # coefficient "one": alpha = 1; "blocks4": log10 alpha ~ U[-6, 6] per 4^d-cell block (seed 0)
    "cfg2_L4h": (2, (2048, 2048), (64, 64), 8, "ve", "cardinality", "uniform", "one", "reference"),
    "cfg2_Lh": (2, (2048, 2048), (64, 64), 32, "ve", "cardinality", "uniform", "one", "reference"),
    "cfg2_L16h": (2, (2048, 2048), (64, 64), 2, "ve", "cardinality", "uniform", "one", "reference"),
    "cfg2_LH": (2, (2048, 2048), (64, 64), 1, "ve", "cardinality", "uniform", "one", "reference"),
    "cfg3": (3, (128, 128, 128), (16, 16, 16), 2, "vef", "cardinality", "one", "one", "reference"),
    # cfg4 runs in spec scaling: with the reference's coarse-basis scaling it does not converge
    # in 2000 iterations
    "cfg4": (3, (128, 128, 128), (16, 16, 16), 2, "vef", "coefficient", "one", "blocks4", "spec"),
    "cfg5": (3, (256, 256, 256), (32, 32, 32), 2, "vef", "cardinality", "uniform", "one", "reference"),
    "cfg1": (2, (64, 64), (4, 4), 4, "ve", "cardinality", "one", "one", "reference"),
}
SAMPLES = {  # bounded CPU samples with the workload's local geometry (subdomain size, split, recipe)
    "cfg2_L4h": [(2, (128, 128), (4, 4), 8), (2, (256, 256), (8, 8), 8)],
    "cfg2_Lh": [(2, (128, 128), (4, 4), 32), (2, (256, 256), (8, 8), 32)],
    "cfg2_L16h": [(2, (128, 128), (4, 4), 2), (2, (256, 256), (8, 8), 2)],
    "cfg2_LH": [(2, (128, 128), (4, 4), 1), (2, (256, 256), (8, 8), 1)],
    "cfg3": [(3, (16, 16, 16), (2, 2, 2), 2), (3, (24, 24, 24), (3, 3, 3), 2), (3, (32, 32, 32), (4, 4, 4), 2)],
    "cfg4": [(3, (16, 16, 16), (2, 2, 2), 2), (3, (24, 24, 24), (3, 3, 3), 2), (3, (32, 32, 32), (4, 4, 4), 2)],
    "cfg5": [(3, (16, 16, 16), (2, 2, 2), 2), (3, (24, 24, 24), (3, 3, 3), 2), (3, (32, 32, 32), (4, 4, 4), 2)],
    "cfg1": [(2, (64, 64), (4, 4), 4)],
}
DESCR = {
    "cfg2": "2D Poisson 2048^2 P1 (4,190,209 dofs), 64x64 subdomains of 32^2 cells, {L} subedges + "
            "vertices ('ve'), cardinality weights, f ~ U[-1,1] (seed 0), rtol 1e-8, reference coarse scaling",
    "cfg3": "3D Poisson 128^3 P1 tets (2,048,383 dofs), 16^3 subdomains of 8^3 cells, 4h subfaces/subedges "
            "+ vertices ('vef'), cardinality weights, f = 1, rtol 1e-8, reference coarse scaling",
    "cfg4": "3D diffusion 128^3 P1 tets, 16^3 subdomains of 8^3, alpha on 4^3-cell blocks with log10 alpha "
            "~ U[-6,6] (seed 0), 4h objects ('vef'), coefficient weights, f = 1, rtol 1e-8, spec coarse scaling",
    "cfg5": "3D Poisson 256^3 P1 tets (16,581,375 dofs), 32^3 subdomains of 8^3 cells, 4h objects ('vef'), "
            "cardinality weights, f ~ U[-1,1] (seed 0), rtol 1e-8, reference coarse scaling",
    "cfg1": "2D Poisson 64^2 P1, 4x4 subdomains of 16^2, L=4h ('ve'), f = 1, rtol 1e-8",
}


def describe(name):
    if name.startswith("cfg2_"):
        return f"{name}: " + DESCR["cfg2"].format(L={"L4h": "L=4h", "Lh": "L=h", "L16h": "L=16h",
                                                     "LH": "L=32h=H"}[name[5:]])
    return f"{name}: " + DESCR[name]


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.nvml = None
        self.lines = []

    def start(self):
        # NVML polling (5 ms period): the cfg2 timed region is ~100 ms, shorter than
        # nvidia-smi's start-up, so nvidia-smi -lms only serves as the fallback
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (N, h)
            self.stop_flag = threading.Event()
            self.ready = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            self.ready.wait(timeout=5)
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def _poll(self):
        N, h = self.nvml
        bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
        mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while not self.stop_flag.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                flags = ["Active" if r & b else "Not Active" for b in bits]
                self.lines.append(", ".join([str(sm), str(mx)] + flags))
            except Exception:
                pass
            self.ready.set()
            time.sleep(0.005)

    def stop(self):
        if self.nvml is not None:
            self.stop_flag.set()
            self.thread.join(timeout=5)
            try:
                self.nvml[0].nvmlShutdown()
            except Exception:
                pass
            return self._summary("nvml")
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        return self._summary("nvidia-smi")

    def _summary(self, source):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": source}


def build_host_problem(name, device=None):
    """The workload's mesh, partition pair, objects, weights, system and rhs; ``device``:
    membership / objects / weights from the device index-set kernels (index_device.py)."""
    import paper_2001_07289_b200 as P

    dim, cells, subs, split, recipe, wmode, source, coef, scaling = WORKLOADS[name]
    t0 = time.perf_counter()
    mesh = P.build_mesh(dim, cells, "p1")
    cf = P.make_constant(mesh, 1.0) if coef == "one" else P.make_blocks(mesh, 4, 0)
    pair = P.refine_uniform(mesh, P.partition_uniform(mesh, subs), split, validate=False)
    objs = P.classify_objects(pair, device=device)
    w = P.compute_weights(pair, wmode, cf, objs)
    system = P.assemble(mesh, cf)
    if source == "uniform":
        b = P.mesh.load_vector(mesh, P.uniform_source(mesh, 0))
    else:
        b = system.rhs
    prep = time.perf_counter() - t0
    return dict(P=P, mesh=mesh, cf=cf, pair=pair, objs=objs, w=w, system=system, b=b,
                recipe=recipe, prep=prep, scaling=scaling)


def phase_work(op, pb, its):
    """Algorithmic bytes / flops per launch of each timed phase on this rank;
    the coarse problem is replicated, so its work is the full problem's on every rank."""
    lay = op.plan.layout
    sl = op.slab  # this rank's subdomains / active rows (everything when unsharded)
    nsub = int(sl.s_hi - sl.s_lo)
    m, nblk, nG, nI = lay.m, lay.nblk, lay.nG, lay.m * lay.nblk
    nc = op.plan.n_con_local[sl.s_lo:sl.s_hi]
    n = int(sl.f_hi - sl.f_lo)
    T = lambda k: k * (k + 1) / 2  # noqa: E731
    w = {}
    # interior solve: packed Linv_j (T(m_pad)) + coupling stencil, forward and backward,
    # + vector gather / scatter (as stored: li_stride doubles per subdomain)
    li = nblk * T(lay.m_pad) + nblk * lay.m_pad * (1 if pb["mesh"].element == "p1" else 3 ** (lay.dim - 1))
    w["apply.bt_solve"] = ("hbm", 8.0 * (2 * nsub * li + 2 * nsub * nI))
    # local Gamma phase 1: q = c Phi^T rho; v = T rho (explicit interface operator, nG_pad^2)
    # runs inside the dataflow coarse solve (its idle CTAs), so its bytes count there
    tbytes = 8.0 * nsub * lay.nG_pad ** 2
    if 256 < lay.nG_pad <= 512:  # T stored and read as its lower triangle (t_lower_only)
        tbytes = 8.0 * nsub * lay.nG_pad * (lay.nG_pad + 1) / 2
    w["apply.gamma1"] = ("hbm", 8.0 * nsub * lay.nG_pad * op.plan.nc_pad)
    w["apply.gamma2"] = ("hbm", 8.0 * nsub * lay.nG_pad * op.plan.nc_pad)
    cp = op.plan.coarse
    if cp is not None:
        w["apply.coarse"] = ("hbm", 8.0 * 2 * cp.factor_entries())
        w["setup.coarse"] = ("fp64", cp.factor_flops())
    if op.stats().tv_in_coarse_solve:
        w["apply.coarse"] = ("hbm", w["apply.coarse"][1] + tbytes)
    else:
        w["apply.gamma1"] = ("hbm", w["apply.gamma1"][1] + tbytes)
    # pcg SpMV + dot: x, y, alpha (cells ~ n)
    w["pcg.spmv_dot"] = ("hbm", 8.0 * 3 * n)
    # setup: E = L_I^{-1} A_IG (block forward, dense n_G RHS), S_G = A_GG - E^T E (SYRK),
    # S_K Cholesky, Phi (TRSMs with n_c RHS, S_C), P = Phi^T S_G Phi
    w["setup.E"] = ("fp64", nsub * (max(nblk - 1, 0) * 2 * m * m * nG + nblk * m * m * nG))
    w["setup.SG"] = ("fp64", nsub * nG * (nG + 1) * nI)
    w["setup.SK"] = ("fp64", nsub * nG**3 / 3)
    ng, ncp = lay.nG_pad, op.plan.nc_pad
    # L^{-1} of the S_K factor (triangular inverse, n^3/3). Phi phase: G = L^{-1} C^T and
    # W = Z C^T are gathers; S_C = G^T G (n nc^2, symmetric), Z = L^{-T} L^{-1} (n^3/3),
    # S_C^{-1} (~nc^3), Phi = W S_C^{-1} (2 n nc^2). T -= Phi W^T (lower: n^2 nc)
    w["setup.Linv"] = ("fp64", nsub * nG**3 / 3)
    w["setup.Phi"] = ("fp64", float(np.sum(nG**3 / 3 + 3 * nG * nc * nc + nc**3)))
    w["setup.T"] = ("fp64", float(np.sum(nG * nG * nc)))
    w["setup.btchol"] = ("fp64", nsub * nblk * (m**3 / 3 + 2 * m**3))
    # fused interior elimination (2D schur2d / 3D schur3d), the formulation's own work: W
    # recursion (Gauss-Jordan inverse of each plane block, 2 m^3) + per plane j with na_j
    # active interface columns: H_j = W_j R_j (2 m^2 na_j) and S_G -= R_j^T H_j (lower half,
    # m na_j^2)
    na = active_prefix(lay)
    w["setup.schur"] = ("fp64", nsub * float(sum(2 * m**3 + 2 * m * m * a + m * a * a for a in na)))
    return w


def active_prefix(lay):
    """Exact active interface prefix per plane (the kernels round it up to 8): one past the
    largest surface slot coupled to an interior node of planes <= j (capi.cu, G.nact)."""
    npd = [b + 1 for b in lay.blk]
    code = lay.node_code
    act = np.zeros(max(lay.nblk, 1), dtype=np.int64)
    coords = np.stack(np.unravel_index(np.arange(lay.nloc_nodes), npd[::-1])[::-1], axis=1)
    interior = np.flatnonzero(code >= 0)
    offs = np.array(np.meshgrid(*[[-1, 0, 1]] * lay.dim, indexing="ij")).reshape(lay.dim, -1).T
    for o in offs:
        nb = coords[interior] + o
        ok = np.all((nb >= 0) & (nb < np.array(npd)), axis=1)
        nbi = np.ravel_multi_index(nb[ok].T[::-1], npd[::-1])
        c = code[nbi]
        surf = c < 0
        planes = code[interior[ok]][surf] // lay.m_pad
        np.maximum.at(act, planes, -c[surf])
    return np.maximum.accumulate(act).tolist()


def _allmax(v, args):
    """Max over ranks (device clock values; CPU tensor for the gloo test transport)."""
    import torch

    dev = "cpu" if args.transport == "host" else "cuda"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2001_07289_b200 import _capi

    torch.cuda.set_device(local_rank)
    torch.zeros(1, device="cuda")  # CUDA context outside the prep timing
    pb = build_host_problem(args.workload, device=local_rank)
    P = pb["P"]
    t0 = time.perf_counter()
    # N > 1: one operator sharded over the ranks (slabs of subdomain rows, NCCL exchanges,
    # replicated coarse problem) — strong scaling of the same global problem
    comm = None
    if world > 1:
        comm = P.HostComm(rank, world) if args.transport == "host" else P.NcclComm(rank, world)
    op = P.build_bddc(pb["system"], pb["pair"], pb["objs"], pb["recipe"], pb["w"],
                      coarse_scaling=pb["scaling"], device=local_rank, comm=comm)
    sl = op.slab
    first_setup_s = time.perf_counter() - t0
    lib = _capi.load()
    ctx = op._ctx
    n = op.n
    b_host = np.ascontiguousarray(pb["b"])
    b_dev = torch.from_numpy(b_host).cuda()
    x_dev = torch.empty_like(b_dev)
    alpha_pin = torch.from_numpy(np.ascontiguousarray(pb["cf"].alpha)).pin_memory()
    b_pin = torch.from_numpy(b_host).pin_memory()
    x_pin = torch.empty(n, dtype=torch.float64).pin_memory()
    tol, maxit = 1e-8, 2000

    def step_device():
        op.refactor()
        return op.pcg(b_dev, tol=tol, max_iters=maxit, x_out=x_dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    # cold one-shot solve right after build_bddc (what experiments.run does once, with the
    # host index sets and first setup before it): reported as cold_e2e
    t1 = time.perf_counter()
    res = op.pcg(b_dev, tol=tol, max_iters=maxit, x_out=x_dev)
    torch.cuda.synchronize()
    cold_solve_s = time.perf_counter() - t1
    for _ in range(args.warmup):
        res = step_device()
    iters = res[4]
    # ---- timed region (device-resident inputs) ----
    sampler = ClockSampler(local_rank)
    lib.bddc_profile(ctx, 1)
    barrier()
    sampler.start()
    l0 = lib.bddc_launch_count()
    lib.bddc_event_record(ctx, 0)
    setup_ms = solve_ms = 0.0
    for _ in range(args.steps):
        lib.bddc_event_record(ctx, 2)
        op.refactor()
        lib.bddc_event_record(ctx, 3)
        res = op.pcg(b_dev, tol=tol, max_iters=maxit, x_out=x_dev)
        lib.bddc_event_record(ctx, 4)
        setup_ms += lib.bddc_event_elapsed_ms(ctx, 2, 3)
        solve_ms += lib.bddc_event_elapsed_ms(ctx, 3, 4)
    lib.bddc_event_record(ctx, 1)
    elapsed = lib.bddc_event_elapsed_ms(ctx, 0, 1)
    launches = lib.bddc_launch_count() - l0
    barrier()
    clocks = sampler.stop()
    phases = {}
    names = ("apply.bt_solve", "apply.gamma1", "apply.coarse", "apply.gamma2", "setup.assemble",
             "setup.schur", "setup.btchol", "setup.E", "setup.SG", "setup.SK", "setup.Linv", "setup.Phi",
             "setup.T", "setup.coarse", "pcg.spmv_dot", "coarse.inverse") + tuple(
                 f"coarse.L{l:02d}" for l in range(20))
    for name in names:
        cnt = C.c_longlong()
        ms = lib.bddc_profile_read(ctx, name.encode(), C.byref(cnt))
        if cnt.value:
            phases[name] = (ms, cnt.value)
    lib.bddc_profile(ctx, 0)
    if world > 1:
        elapsed = _allmax(elapsed, args)
    x, alphas, betas, hist, k, conv = res
    kappa = None
    try:
        from paper_2001_07289_b200.krylov import _lanczos_extremes

        lo, hi = _lanczos_extremes(list(alphas), list(betas))
        kappa = hi / lo
    except Exception:
        pass

    # ---- e2e through the C ABI with host buffers ----
    err = C.create_string_buffer(512)
    rep = _capi.PcgReport()
    al = np.zeros(maxit + 1)
    be = np.zeros(maxit + 1)
    rs = np.zeros(maxit + 2)
    pd = C.POINTER(C.c_double)

    def step_e2e():  # setup + solve from host buffers (alpha, b up; x down) in one C-ABI call
        rc = lib.bddc_solve_host(ctx, C.cast(alpha_pin.data_ptr(), pd), C.cast(b_pin.data_ptr(), pd),
                                 C.cast(x_pin.data_ptr(), pd), tol, maxit, _capi.ptr(al, C.c_double),
                                 _capi.ptr(be, C.c_double), _capi.ptr(rs, C.c_double), C.byref(rep),
                                 err, len(err))
        assert rc == 0, err.value

    for _ in range(max(1, min(args.warmup, 2))):
        step_e2e()
    barrier()
    lib.bddc_event_record(ctx, 5)
    for _ in range(args.steps):
        step_e2e()
    lib.bddc_event_record(ctx, 6)
    e2e_ms = lib.bddc_event_elapsed_ms(ctx, 5, 6)
    barrier()
    if world > 1:
        e2e_ms = _allmax(e2e_ms, args)
    own = slice(sl.fo_lo, sl.fo_hi)  # sharded: this rank's rows of x
    xe2e = x_pin.numpy()[own].copy()
    e2e_consistent = float(np.linalg.norm(xe2e - x_dev.cpu().numpy()[own]) / np.linalg.norm(xe2e))
    if world > 1:
        e2e_consistent = _allmax(e2e_consistent, args)

    # ---- host link probe (explains e2e - value): one b-sized copy each way, CUDA events ----
    pcie = None
    try:
        cs = torch.cuda.Stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs):
            e0.record(cs)
            b_dev.copy_(b_pin, non_blocking=True)
            e1.record(cs)
        cs.synchronize()
        h2d = b_pin.numel() * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9
        with torch.cuda.stream(cs):
            e0.record(cs)
            x_pin.copy_(x_dev, non_blocking=True)
            e1.record(cs)
        cs.synchronize()
        d2h = x_pin.numel() * 8 / (e0.elapsed_time(e1) * 1e-3) / 1e9
        pcie = {"h2d_gbs": round(h2d, 1), "d2h_gbs": round(d2h, 1), "bytes": int(b_pin.numel() * 8)}
    except Exception:
        pcie = None

    # ---- preconditioner applies/s (device-resident r) ----
    r = torch.from_numpy(np.random.default_rng(1).standard_normal(n)).cuda()
    z = torch.empty_like(r)
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        lib.bddc_apply(ctx, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()), C.c_void_p(stream))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    napp = 50
    e0.record()
    for _ in range(napp):
        lib.bddc_apply(ctx, C.c_void_p(r.data_ptr()), C.c_void_p(z.data_ptr()), C.c_void_p(stream))
    e1.record()
    torch.cuda.synchronize()
    apply_ms = e0.elapsed_time(e1) / napp

    # ---- rooflines per phase ----
    hbm, hbm_src = _peaks()
    work = phase_work(op, pb, k)
    if op.stats().t_in_coarse_factor and "setup.coarse" in work and "setup.T" in work:
        # the local T tiles ran inside the dataflow coarse factorization
        work["setup.coarse"] = ("fp64", work["setup.coarse"][1] + work["setup.T"][1])
    phase_out = {}
    for name, (ms, cnt) in phases.items():
        kind, amount = work.get(name, (None, None))
        avg = ms / cnt
        if kind and name.startswith("setup.") and cnt > args.steps:
            amount = amount * args.steps / cnt  # setup phase in several subdomain chunks per step
        entry = {"ms_total": round(ms, 3), "launches": cnt, "avg_ms": round(avg, 4)}
        if kind == "hbm":
            ach = amount / (avg * 1e-3) / 1e9
            entry.update(bound="hbm", achieved=round(ach, 1), unit="GB/s", frac=round(ach / hbm, 4))
        elif kind == "fp64":
            ach = amount / (avg * 1e-3) / 1e12
            entry.update(bound="fp64", achieved=round(ach, 3), unit="TFLOP/s",
                         frac=round(ach / FP64_PEAK_TFLOPS, 4))
        phase_out[name] = entry
    dominant = max(phase_out, key=lambda k2: phase_out[k2]["ms_total"]) if phase_out else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath) and dominant:
        try:
            traffic = json.load(open(tpath)).get(args.workload, {}).get(dominant)
        except Exception:
            traffic = None
    roof = None
    if dominant:
        d = phase_out[dominant]
        roof = {"kernel": dominant, "bound": "hbm" if d.get("bound") == "hbm" else "tensor",
                "pipe": "HBM3e stream" if d.get("bound") == "hbm" else
                "FP64 tensor pipe: DMMA.8x8x4 via mma.sync (tcgen05 has no f64 kind on sm_100a)",
                "achieved": d.get("achieved"), "unit": d.get("unit"),
                "peak": hbm if d.get("bound") == "hbm" else FP64_PEAK_TFLOPS,
                "peak_source": hbm_src if d.get("bound") == "hbm" else
                "measured cuBLAS FP64 GEMM (no FP64 entry in MEASURED_PEAKS.json)",
                "frac": d.get("frac"), "traffic": traffic}

    # ---- CPU baseline (oracle port, bounded sample, rank 0) ----
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.workload)

    nsteps = args.steps
    value = n * nsteps / (elapsed * 1e-3) / 1e6  # one global problem over all ranks
    e2e_val = n * nsteps / (e2e_ms * 1e-3) / 1e6
    # host<->device bytes per step over all ranks: alpha + the active rows of b in, owned x out
    ncell = len(pb["cf"].alpha)
    h2d = sum(8 * ncell + 8 * (s2.f_hi - s2.f_lo) for s2 in (
        P.slab_ranges(pb["mesh"].dim, pb["mesh"].cells_per_dim, pb["pair"].box_layout[0], r2, world)
        for r2 in range(world)))
    d2h = 8 * n + world * 8 * 4 * (k + 1)
    st = op.stats()
    line = {
        "metric": "BDDC-SO setup+PCG solve throughput (Mdof/s)",
        "value": round(value, 3),
        "unit": "Mdof/s",
        "n_gpus": world,
        "steps": nsteps,
        "warmup": args.warmup,
        "ms_per_step": round(elapsed / nsteps, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded f / alpha as in config.workload)",
        "config": {
            "workload": describe(args.workload),
            "dofs": n, "subdomains": int(st.nsub), "coarse_size": int(st.n_coarse),
            "parallelism": "single GPU" if world == 1 else
                           f"sharded x{world}: slabs of subdomain rows along the last axis, "
                           + ("host-staged (gloo, ranks sharing one GPU: test transport)" if args.transport == "host"
                              else "NCCL") + " halo / allgather exchanges, "
                           + ("replicated coarse problem" if os.environ.get("BDDC_DIST_COARSE") == "0" else
                              "coarse ND subtrees per rank + replicated top (DESIGN.md §9.2)"),
            "l2": "inputs > L2 (factors %.1f GB + fronts %.2f GB vs 126 MB L2)" % (
                st.factor_bytes / 1e9, st.front_bytes / 1e9),
        },
        "e2e": {"value": round(e2e_val, 3), "unit": "Mdof/s",
                "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "ms_per_step": round(e2e_ms / nsteps, 3),
                "x_matches_device_run": e2e_consistent < 1e-14,
                "overlap": "alpha (slabs of subdomain rows) and b uploads overlap the setup; x download after the solve",
                "host_link": pcie},
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clocks,
        "gpu_launches": int(launches),
        "iterations": int(k),
        "converged": bool(conv),
        "kappa": kappa,
        "setup_ms": round(setup_ms / nsteps, 3),
        "solve_ms": round(solve_ms / nsteps, 3),
        "applies_per_s": round(1000.0 / apply_ms, 1),
        "apply_ms": round(apply_ms, 4),
        "prep_s": round(pb["prep"] + op.times.prep_s, 2),  # + build_bddc host tables
        "first_setup_s": round(first_setup_s, 2),
        "cold_e2e": {
            "value": round(n / (pb["prep"] + first_setup_s + cold_solve_s) / 1e6, 4), "unit": "Mdof/s",
            "prep_s": round(pb["prep"], 2), "first_setup_s": round(first_setup_s, 2),
            "solve_s": round(cold_solve_s, 3),
            "what": "one-shot through the Python API from nothing: mesh / partition / objects / weights "
                    "(prep_s), build_bddc incl. its index tables, symbolic analysis and first numeric setup "
                    "(first_setup_s), one pcg (solve_s)"},
        "phases": phase_out,
    }
    op.close()
    if rank == 0 and world == 1 and args.workload == "cfg5" and not args.no_three_level:
        line["three_level"] = three_level_extra(args.workload)
    if rank == 0:
        print(json.dumps(line), flush=True)


def three_level_extra(workload):
    """Extra field of the cfg5 line: the three-level BDDC-SO prototype on the same
    workload, run by tools/three_level_bench.py in a child process after this process released
    its operator (a failure there cannot touch the line). It is the paper's outlook, NOT the
    reference's method (more iterations, another preconditioner), so it is excluded from
    value / e2e / roofline and only reported next to them."""
    import subprocess

    import torch

    try:
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        env = dict(os.environ, PYTORCH_CUDA_ALLOC_CONF="expandable_segments:True")
        p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "three_level_bench.py"), "--workload",
                            workload, "--coarsening", "2", "--lean"], capture_output=True, text=True,
                           timeout=420, env=env)
        if p.returncode:
            return {"unavailable": ("exit %d: " % p.returncode) + p.stderr.strip().splitlines()[-1][:200]}
        d = json.loads(p.stdout.strip().splitlines()[-1])
        return {"note": "three-level BDDC-SO prototype (paper's outlook; not the reference's method: excluded "
                        "from value / e2e / roofline), one re-setup + PCG to the same rtol, set up without a "
                        "coarse factorization",
                "value": d["Mdof_s"], "unit": "Mdof/s", "ms_per_step": d["step_ms"],
                "setup_ms": d["refactor_ms"], "solve_ms": d["pcg_ms"], "iterations": d["iterations"],
                "kappa": d["kappa"], "true_residual_rel": d["true_residual_rel"],
                "level2": d["level2"], "cold_build_s": d["cold_build_s"],
                "gpu_memory_used_gb": d["gpu_memory_used_gb"]}
    except Exception as e:  # noqa: BLE001 - an optional extra must never cost the line
        return {"unavailable": str(e)[:200]}


def _sample_alpha(cells, coef):
    from oracle import bddc_oracle as orc

    return None if coef == "one" else orc.block_alpha(cells, 4, 0)


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_worker(args):
    """One CPU process of the baseline (spawned by cpu_measure with 1-thread BLAS): prep +
    warm-up, then 'ready'; on 'go' it times --steps steps of build_bddc's numeric work
    (oracle _build: per-subdomain SuperLU factorizations, Psi, coarse assembly + SuperLU;
    bddc.py:393-523) + pcg to rtol 1e-8 (krylov.py:31-92) and prints one JSON line."""
    from oracle import bddc_oracle as orc

    dim, cells, subs, split = SAMPLES[args.workload][args.cpu_sample]
    _, _, _, _, recipe, wmode, source, coef, scaling = WORKLOADS[args.workload]
    o = orc.Oracle(dim, cells, subs, split, recipe, wmode, "p1", _sample_alpha(cells, coef), scaling)
    mesh = o.mesh
    b = orc.load(mesh, orc.uniform_f(mesh.n_free, 0)) if source == "uniform" else orc.load(mesh, 1.0)

    def step():
        t0 = time.perf_counter()
        o._build()
        t1 = time.perf_counter()
        x, rep = orc.pcg(o.matvec, o.apply, b, 1e-8, 2000)
        return t1 - t0, time.perf_counter() - t1, rep["iterations"]

    for _ in range(args.warmup):
        step()
    print("ready", flush=True)
    sys.stdin.readline()
    res = [step() for _ in range(args.steps)]
    print(json.dumps({"n": int(mesh.n_free), "build": [r[0] for r in res], "pcg": [r[1] for r in res],
                      "its": res[-1][2]}), flush=True)


def cpu_measure(workload, sample, steps, warmup, procs=None):
    """The reference algorithm (oracle port) on the host: `procs` concurrent processes (all
    host cores by default), each with single-threaded BLAS (OpenBLAS threads on these small
    SuperLU / BLAS calls are 5-8x slower than one thread: measured), each solving its own
    copy of the bounded sample `sample` of `workload` for `steps` timed steps after `warmup`.
    The processes start the timed steps together; value = dofs solved by all of them / wall
    time. One routine for both the cpu_baseline field and --impl reference."""
    procs = procs or _host_cores()
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1")
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-worker", "--workload", workload,
           "--cpu-sample", str(sample), "--steps", str(steps), "--warmup", str(warmup)]
    ps = [subprocess.Popen(cmd, stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True, env=env)
          for _ in range(procs)]
    try:
        for p in ps:
            if p.stdout.readline().strip() != "ready":
                raise RuntimeError("CPU baseline worker failed")
        t0 = time.perf_counter()
        for p in ps:
            p.stdin.write("go\n")
            p.stdin.flush()
        outs = [json.loads(p.stdout.readline()) for p in ps]
        wall = time.perf_counter() - t0
    finally:
        for p in ps:
            try:
                p.stdin.close()
            except Exception:
                pass
            p.wait(timeout=60)
    n = outs[0]["n"]
    dim, cells, subs, split = SAMPLES[workload][sample]
    build = statistics.median(t for o in outs for t in o["build"])
    pcg = statistics.median(t for o in outs for t in o["pcg"])
    return {"value": procs * n * steps / wall / 1e6, "dofs": n, "procs": procs, "wall_s": wall,
            "build_s": build, "pcg_s": pcg, "its": outs[0]["its"],
            "sample": f"{dim}D {cells} P1, {subs} subdomains of the workload's local geometry "
                      f"(split {split}), {n} dofs"}


def _cpu_line(m, trend=None):
    cores = m["procs"]
    d = {"value": round(m["value"], 5), "unit": "Mdof/s", "cores": cores, "kind": "port",
         "cpu_model": _cpu_model(), "threads": f"{cores} processes x 1 BLAS thread (OPENBLAS_NUM_THREADS=1)",
         "sample": (f"{m['sample']}; {cores} concurrent copies, each setup (build_bddc numeric) "
                    f"{m['build_s']:.3f} s + pcg {m['pcg_s']:.3f} s ({m['its']} its), median over steps")}
    if trend:
        d["trend"] = trend
    return d


def cpu_baseline(workload):
    """cpu_baseline field (rank 0, N=1): every bounded sample of the workload (smallest
    first) so the per-dof trend toward the full config is visible; value = the largest."""
    trend, last = [], None
    for i in range(len(SAMPLES[workload])):
        m = cpu_measure(workload, i, steps=2, warmup=1)
        trend.append({"dofs": m["dofs"], "Mdof_s": round(m["value"], 5),
                      "setup_s": round(m["build_s"], 4), "pcg_s": round(m["pcg_s"], 4)})
        last = m
    return _cpu_line(last, trend)


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU algorithm (oracle port, pinned to the reference
    by tests/golden) on the host cores, same routine as cpu_baseline, largest sample."""
    if rank != 0:
        return
    m = cpu_measure(args.workload, len(SAMPLES[args.workload]) - 1, args.steps, args.warmup)
    value = m["value"]
    cpu = _cpu_line(m)
    line = {
        "metric": "BDDC-SO setup+PCG solve throughput (Mdof/s)", "value": round(value, 5),
        "unit": "Mdof/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * m["wall_s"] / args.steps, 2), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": describe(args.workload), "sample": cpu["sample"]}, "impl": "reference",
        "cpu_baseline": cpu,
        "e2e": {"value": round(value, 5), "unit": "Mdof/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "iterations": m["its"],
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-three-level", action="store_true",
                    help="skip the three-level extra field of the cfg5 line (DESIGN.md §10a)")
    ap.add_argument("--cpu-worker", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-sample", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--transport", default="nccl", choices=("nccl", "host"),
                    help="host: test-only gloo + host-staged exchanges with every rank on cuda:0")
    args = ap.parse_args()
    if args.cpu_worker:
        cpu_worker(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch

        if args.transport == "host":
            local_rank = 0
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.distributed.init_process_group("gloo" if args.transport == "host" else "nccl")
    run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch

        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
