"""Index sets on the GPU: membership, interface objects, counting / cardinality weights.

Host side of ``csrc/index_sets.cu`` (C ABI ``bddc_index_*``), SURVEY §8(f)2. It replaces the
reference's host index-set code for a partition pair:

* ``_node_membership`` / Γ, Γ̂        partition.py:75-83, 117-131
* ``classify_objects``                partition.py:223-250
* ``compute_weights`` counting and cardinality modes   bddc.py:108-145

and returns the same objects the host statement (partition.py / weights.py here) returns,
bit-identical (tests/test_index_device.py checks both against the reference fixtures). The
coefficient weighting needs exact rational sums of α (bddc.py:137-142) and stays on the host.
The per-dof membership tuples (``on_gamma`` …) are only materialised, on the host, if a
caller asks for them; the device path itself never needs them.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _capi
from .partition import MembershipSets, ObjectTable, PartitionPair, _host_membership


class DeviceMembership:
    """``pair.membership`` after a device classification: Γ and Γ̂ from the device; the
    per-dof tuple tables (on_gamma, on_gamma_hat, *_rows, *_counts) built on first access."""

    def __init__(self, pair: PartitionPair, gamma_dofs: np.ndarray, gamma_hat_dofs: np.ndarray):
        self._pair = pair
        self.gamma_dofs = gamma_dofs
        self.gamma_hat_dofs = gamma_hat_dofs
        self._full: MembershipSets | None = None

    def _host(self) -> MembershipSets:
        if self._full is None:
            self._full = _host_membership(self._pair)
        return self._full

    def __getattr__(self, name):
        if name in ("on_gamma", "on_gamma_hat", "theta_rows", "theta_counts", "hat_rows", "hat_counts"):
            return getattr(self._host(), name)
        raise AttributeError(name)


def _raise(rc: int, err) -> None:
    if rc == 1:
        raise ValueError(err.value.decode(errors="replace") or "invalid argument")
    if rc:
        raise RuntimeError("CUDA error in the device index sets: " + err.value.decode(errors="replace"))


def device_index_sets(pair: PartitionPair, device: int = 0) -> dict:
    """Run the device pipeline; returns numpy arrays keyed like the C ABI names."""
    lib = _capi.load()
    mesh = pair.mesh
    dim = mesh.dim
    cells = np.zeros(3, dtype=np.int32)
    cells[:dim] = mesh.cells_per_dim
    hat = np.ascontiguousarray(pair.theta_hat, dtype=np.int32)
    parent = np.ascontiguousarray(pair.parent, dtype=np.int32)
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    rc = lib.bddc_index_build(int(device), dim, _capi.ptr(cells, C.c_int), _capi.ptr(hat, C.c_int),
                              _capi.ptr(parent, C.c_int), int(len(parent)), C.byref(h), err, len(err))
    _raise(rc, err)
    try:
        size = {k: int(lib.bddc_index_size(h, k.encode())) for k in
                ("n_free", "n_gamma", "n_gamma_hat", "n_obj", "width")}
        W, n_obj, n_gamma = size["width"], size["n_obj"], size["n_gamma"]
        shapes = {
            "gamma_dofs": (n_gamma, np.int64), "gamma_hat_dofs": (size["n_gamma_hat"], np.int64),
            "signature": (n_obj * W, np.int64), "sig_len": (n_obj, np.int64),
            "owners": (n_obj * W, np.int64), "owner_len": (n_obj, np.int64),
            "dof_ptr": (n_obj + 1, np.int64), "dof_list": (n_gamma, np.int64),
            "dof_obj": (size["n_free"], np.int64), "card_counts": (n_obj * W, np.int64),
            "kind": (n_obj, np.int8), "w_counting": (n_obj * W, np.float64),
            "w_cardinality": (n_obj * W, np.float64),
        }
        out = {}
        for name, (n, dt) in shapes.items():
            a = np.empty(n, dtype=dt)
            if lib.bddc_index_copy(h, name.encode(), C.c_void_p(a.ctypes.data), int(n)):
                raise RuntimeError(f"device index sets: copy of {name} failed")
            out[name] = a
        for name in ("signature", "owners", "card_counts", "w_counting", "w_cardinality"):
            out[name] = out[name].reshape(n_obj, W)
        out.update(size)
        return out
    finally:
        lib.bddc_index_free(h)


def classify_objects_device(pair: PartitionPair, device: int = 0) -> ObjectTable:
    """``classify_objects`` on the GPU; also installs the device membership on ``pair`` and
    keeps the counting / cardinality object weights for ``compute_weights``."""
    r = device_index_sets(pair, device)
    pair.__dict__["membership"] = DeviceMembership(pair, r["gamma_dofs"], r["gamma_hat_dofs"])
    t = ObjectTable(pair.mesh.dim, r["signature"], r["sig_len"], r["owners"], r["owner_len"], r["kind"],
                    r["dof_ptr"], r["dof_list"], r["dof_obj"])
    t._device_weights = {"counting": (r["w_counting"], None),
                         "cardinality": (r["w_cardinality"], r["card_counts"])}
    return t


__all__ = ["DeviceMembership", "classify_objects_device", "device_index_sets"]
