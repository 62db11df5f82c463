"""Multi-GPU sharding on CPU: the slab partition (Python restatement vs the
library's host function), its invariants, and the sharded apply emulated by world-size-2
gloo ranks that exchange exactly what the library exchanges (poisoned elsewhere)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import build_problem, load_golden
from paper_2001_07289_b200 import _capi, slab_ranges


def _lib_slab(dim, cells, subs, rank, world):
    lib = _capi.load()
    out = (C.c_longlong * 10)()
    ce = (C.c_int * 3)(*(list(cells) + [1] * (3 - dim)))
    su = (C.c_int * 3)(*(list(subs) + [1] * (3 - dim)))
    rc = lib.bddc_partition_info(dim, ce, su, rank, world, out)
    return rc, list(out)


BOXES = [(2, (64, 64), (4, 4)), (2, (32, 32), (4, 4)), (3, (32, 32, 32), (4, 4, 4)),
         (2, (2048, 2048), (64, 64)), (3, (128, 128, 128), (16, 16, 16)), (2, (96, 60), (3, 5))]


@pytest.mark.parametrize("dim,cells,subs", BOXES)
def test_partition_matches_library(dim, cells, subs):
    for world in range(1, min(subs[dim - 1], 8) + 1):
        for rank in range(world):
            rc, out = _lib_slab(dim, cells, subs, rank, world)
            s = slab_ranges(dim, cells, subs, rank, world)
            assert rc == 0
            assert out == [s.s_lo, s.s_hi, s.f_lo, s.f_hi, s.fo_lo, s.fo_hi, s.lo_send, s.lo_recv,
                           s.hi_send, s.hi_recv]


@pytest.mark.parametrize("dim,cells,subs", BOXES)
def test_partition_invariants(dim, cells, subs):
    n = int(np.prod([c - 1 for c in cells]))
    nsub = int(np.prod(subs))
    for world in range(1, min(subs[dim - 1], 8) + 1):
        sl = [slab_ranges(dim, cells, subs, r, world) for r in range(world)]
        # subdomains and owned dofs are partitioned, in rank order
        assert [s.s_lo for s in sl][0] == 0 and sl[-1].s_hi == nsub
        assert all(a.s_hi == b.s_lo for a, b in zip(sl, sl[1:]))
        assert sl[0].fo_lo == 0 and sl[-1].fo_hi == n
        assert all(a.fo_hi == b.fo_lo for a, b in zip(sl, sl[1:]))
        for r, s in enumerate(sl):
            assert s.f_lo <= s.fo_lo < s.fo_hi == s.f_hi
            # halo rows received are owned by the neighbour, rows sent are owned here
            if r > 0:
                assert sl[r - 1].fo_lo <= s.lo_recv and s.lo_recv + s.row_len <= sl[r - 1].fo_hi
                assert s.fo_lo <= s.lo_send and s.lo_send + s.row_len <= s.fo_hi
                assert s.lo_recv + s.row_len <= s.f_lo  # just below the active rows
            if r < world - 1:
                assert sl[r + 1].fo_lo <= s.hi_recv and s.hi_recv + s.row_len <= sl[r + 1].fo_hi
                assert s.hi_recv == s.f_hi  # just above the active rows
    with pytest.raises(ValueError):
        slab_ranges(dim, cells, subs, 0, subs[dim - 1] + 1)
    assert _lib_slab(dim, cells, subs, 0, subs[dim - 1] + 1)[0] == 1


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case):
    import torch.distributed as dist

    from device_emulator import Emulator
    from paper_2001_07289_b200 import select_constraints
    from paper_2001_07289_b200.layout import build_device_plan
    from sharded_emulator import GlooExchange, sharded_apply

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden(case)
        pb = build_problem(g)
        cons = select_constraints(pb["objects"], pb["recipe"], pb["pair"])
        plan = build_device_plan(pb["pair"], cons, pb["weights"])
        em = Emulator(pb["system"], pb["pair"], plan, pb["mode"])
        mesh = pb["mesh"]
        subs = pb["pair"].box_layout[0]
        slabs = [slab_ranges(mesh.dim, mesh.cells_per_dim, subs, r, world) for r in range(world)]
        sl = slabs[rank]
        z = sharded_apply(em, plan, g["r"], sl, slabs, GlooExchange(rank, world))
        ref = em.apply(g["r"])
        act = slice(sl.f_lo, sl.f_hi)
        assert np.isfinite(z[act]).all(), "a value needed on this rank was never exchanged"
        scale = np.abs(ref).max()
        assert np.abs(z[act] - ref[act]).max() <= 1e-14 * scale
        tol = 1e-9 if "cfg4" in case else 1e-12
        own = slice(sl.fo_lo, sl.fo_hi)
        assert np.abs(z[own] - g["Br"][own]).max() <= tol * np.abs(g["Br"]).max()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,world", [("cfg1_p1_ref", 2), ("full_p1_2d", 2), ("cfg3a_p1_ref", 2),
                                        ("cfg1_q1_ref", 3)])
def test_sharded_apply_gloo(case, world):
    mp.spawn(_worker, args=(world, _free_port(), case), nprocs=world, join=True)
