"""Multi-GPU sharding of the operator: one rank per GPU, slabs of the
subdomain lattice along the last axis.

``slab_ranges`` restates the library's partition (csrc/multigpu.cu ``slab_partition``) for
host-side use and CPU tests. ``NcclComm`` / ``HostComm`` attach a rank to a device operator
before its setup:

* ``NcclComm``: the library's own NCCL communicator (unique id broadcast through
  ``torch.distributed``); exchanges run on the operator stream between kernels.
* ``HostComm``: exchanges staged through host buffers and carried by ``torch.distributed``
  (gloo) — for ranks that share one GPU in tests, where NCCL cannot run.

The reference is a single process (bddc.py:419-511 loops over all subdomains); a sharded
operator computes the same preconditioner: every rank factors its own subdomains and
keeps a replicated coarse problem assembled in the single-rank order.
"""

from __future__ import annotations

import ctypes as C
import traceback
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Slab:
    s_lo: int       # subdomains [s_lo, s_hi)
    s_hi: int
    f_lo: int       # active free dofs [f_lo, f_hi): node rows from the lower to the upper cut
    f_hi: int
    fo_lo: int      # owned free dofs (cut line -> lower rank)
    fo_hi: int
    lo_send: int    # halo rows (free-dof offsets of one row / plane), -1 = no neighbour
    lo_recv: int
    hi_send: int
    hi_recv: int
    row_len: int
    sub_row: int


def slab_ranges(dim: int, cells, subs, rank: int, world: int) -> Slab:
    """Slab of ``rank`` (mirrors csrc/multigpu.cu slab_partition)."""
    cells = [int(c) for c in cells][:dim]
    subs = [int(s) for s in subs][:dim]
    ax = dim - 1
    R = subs[ax]
    if not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    if world > R:
        raise ValueError(f"more ranks ({world}) than subdomain rows along the last axis ({R})")
    blk = [c // s for c, s in zip(cells, subs)]
    if world > 1 and blk[ax] < 2:
        raise ValueError("sharding needs >= 2 cells per subdomain along the last axis")
    nfree = [c - 1 for c in cells]
    n = int(np.prod(nfree))
    nsub = int(np.prod(subs))
    r_lo, r_hi = rank * R // world, (rank + 1) * R // world
    sub_row = nsub // R
    row_len = n // nfree[ax]
    H = blk[ax]
    cut_lo, cut_hi = r_lo * H, r_hi * H
    y_lo, y_hi = max(cut_lo, 1), min(cut_hi, cells[ax] - 1)
    f_lo, f_hi = (y_lo - 1) * row_len, y_hi * row_len
    fo_lo = f_lo if rank == 0 else cut_lo * row_len
    lo_send = lo_recv = hi_send = hi_recv = -1
    if rank > 0:
        lo_recv, lo_send = (cut_lo - 2) * row_len, cut_lo * row_len
    if rank < world - 1:
        hi_recv, hi_send = cut_hi * row_len, (cut_hi - 2) * row_len
    return Slab(r_lo * sub_row, r_hi * sub_row, f_lo, f_hi, fo_lo, f_hi, lo_send, lo_recv,
                hi_send, hi_recv, row_len, sub_row)


EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.POINTER(C.c_double),
                          C.POINTER(C.c_double), C.c_longlong, C.c_int)


class NcclComm:
    """Attach the operator to an NCCL communicator of ``world`` ranks (one GPU each)."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group

    def attach(self, lib, ctx):
        import torch.distributed as dist

        uid = C.create_string_buffer(128)
        if self.rank == 0 and lib.bddc_nccl_unique_id(uid) != 0:
            raise RuntimeError("ncclGetUniqueId failed")
        obj = [bytes(uid.raw) if self.rank == 0 else None]
        if self.world > 1:
            dist.broadcast_object_list(obj, src=0, group=self.group)
        buf = C.create_string_buffer(obj[0], 128)
        rc = lib.bddc_comm_init_nccl(ctx, self.rank, self.world, buf)
        if rc:
            raise RuntimeError(f"bddc_comm_init_nccl failed ({rc})")


class HostComm:
    """Exchanges through host buffers over ``torch.distributed`` (gloo): test transport."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group
        self._fn = EXCHANGE_FN(self._exchange)  # keep the thunk alive

    def _exchange(self, user, op, a, b, n, peer):
        try:
            import torch
            import torch.distributed as dist

            ta = torch.from_numpy(np.ctypeslib.as_array(a, shape=(n,)))
            if op == 1:
                tb = torch.from_numpy(np.ctypeslib.as_array(b, shape=(n,)))
                reqs = [dist.isend(ta.clone(), peer, group=self.group),
                        dist.irecv(tb, peer, group=self.group)]
                for r in reqs:
                    r.wait()
            elif op == 2:
                dist.broadcast(ta, src=peer, group=self.group)
            elif op == 3:
                dist.all_reduce(ta, op=dist.ReduceOp.SUM, group=self.group)
            elif op == 4:
                dist.all_reduce(ta, op=dist.ReduceOp.MAX, group=self.group)
            else:
                return 1
            return 0
        except Exception:  # noqa: BLE001 - reported to the library as a failed exchange
            traceback.print_exc()
            return 1

    def attach(self, lib, ctx):
        rc = lib.bddc_comm_init_host(ctx, self.rank, self.world, self._fn, None)
        if rc:
            raise RuntimeError(f"bddc_comm_init_host failed ({rc})")


__all__ = ["Slab", "slab_ranges", "NcclComm", "HostComm"]
