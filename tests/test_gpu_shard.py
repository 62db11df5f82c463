"""Sharded operator on the GPU: world-size-2/3 ranks as processes sharing one
GPU, exchanging through the host-callback transport over gloo (NCCL needs one GPU per
rank; the exchange points and every range-restricted kernel are the same). Each rank's
owned rows of B r, and the gathered PCG solution, must match the single-process fixtures."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import build_problem, load_golden

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case):
    import torch.distributed as dist

    import paper_2001_07289_b200 as P

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden(case)
        pb = build_problem(g)
        op = P.build_bddc(pb["system"], pb["pair"], pb["objects"], pb["recipe"], pb["weights"],
                          coarse_scaling=pb["mode"], comm=P.HostComm(rank, world))
        sl = op.slab
        z = op.apply(g["r"])
        own = slice(sl.fo_lo, sl.fo_hi)
        tol = 1e-9 if "cfg4" in case else 1e-12
        assert np.abs(z[own] - g["Br"][own]).max() <= tol * np.abs(g["Br"]).max()
        x, rep = P.pcg(op.matvec, op.apply, g["b"], tol=float(g["tol"]), max_iters=2000)
        assert abs(rep.iterations - int(g["iterations"])) <= 1
        assert abs(rep.kappa_estimate - float(g["kappa"])) <= 1e-6 * float(g["kappa"])
        assert np.linalg.norm(x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])
        op.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("cfg1_p1_ref", 2), ("cfg3a_p1_ref", 2), ("cfg2a_p1_L4h", 3),
                                        ("full_p1_2d", 4), ("cfg3c_p1_ref", 2), ("cfg3c_p1_ref", 4),
                                        ("cfg4a_p1_spec", 2)])
def test_sharded_operator_matches_fixtures(cuda_ok, case, world):
    """Distributed coarse factorization (each rank factors and solves its ND subtrees, the top
    is replicated: DESIGN.md §9.2) on every case whose tree is deep enough."""
    mp.spawn(_worker, args=(world, _free_port(), case), nprocs=world, join=True)


@pytest.mark.parametrize("case,world", [("cfg3a_p1_ref", 2), ("cfg2a_p1_L4h", 3)])
def test_sharded_operator_replicated_coarse(cuda_ok, case, world, monkeypatch):
    """BDDC_DIST_COARSE=0: every rank factors the whole coarse problem (the round-1 path)."""
    monkeypatch.setenv("BDDC_DIST_COARSE", "0")
    mp.spawn(_worker, args=(world, _free_port(), case), nprocs=world, join=True)


def _nccl_worker(rank, world, port, case):
    """One rank per GPU with the NCCL transport (bddc_comm_init_nccl): the production path."""
    import torch
    import torch.distributed as dist

    import paper_2001_07289_b200 as P

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # plumbing for the NCCL unique id
    try:
        g = load_golden(case)
        pb = build_problem(g)
        op = P.build_bddc(pb["system"], pb["pair"], pb["objects"], pb["recipe"], pb["weights"],
                          coarse_scaling=pb["mode"], device=rank, comm=P.NcclComm(rank, world))
        sl = op.slab
        z = op.apply(g["r"])
        own = slice(sl.fo_lo, sl.fo_hi)
        assert np.abs(z[own] - g["Br"][own]).max() <= 1e-12 * np.abs(g["Br"]).max()
        x, rep = P.pcg(op.matvec, op.apply, g["b"], tol=float(g["tol"]), max_iters=2000)
        assert abs(rep.iterations - int(g["iterations"])) <= 1
        assert np.linalg.norm(x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])
        op.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["cfg3a_p1_ref", "cfg2a_p1_L4h"])
def test_nccl_transport_two_gpus(cuda_ok, case):
    """The NCCL transport over two GPUs (skipped on a one-GPU box: NCCL needs a GPU per rank)."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    mp.spawn(_nccl_worker, args=(2, _free_port(), case), nprocs=2, join=True)


def test_nccl_binding_selftest_one_gpu(cuda_ok):
    """Every NCCL symbol the transport binds (dlopen of the process's libnccl, CommInitRank,
    AllReduce sum / max, grouped Broadcast, grouped Send/Recv) runs once on a world-1
    communicator on this GPU: the one part of the NCCL path a one-GPU box can execute."""
    import torch  # noqa: F401 - loads torch's NCCL first, as a sharded run does

    from paper_2001_07289_b200 import _capi

    assert _capi.load().bddc_nccl_selftest(0) == 0
