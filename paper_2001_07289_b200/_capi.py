"""ctypes binding of the C ABI in include/bddcso_b200.h (libbddcso_b200.so, built in-tree).

There is no fallback: if the CUDA library is missing or no GPU is present, the device
operator raises. This is the binding a reference-side maintainer would add.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BDDC_LIB") or os.path.join(_HERE, "libbddcso_b200.so")  # BDDC_LIB: A/B builds (tools)

_i = C.c_int
_ll = C.c_longlong
_d = C.c_double
_pi = C.POINTER(C.c_int)
_pll = C.POINTER(C.c_longlong)
_pd = C.POINTER(C.c_double)
_vp = C.c_void_p

# coarse-solver hook of the multilevel operator: (user, rhs_dev, sol_dev, n_coarse, stream) -> rc
COARSE_SOLVER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p)

EXPORTS = (
    "bddc_create", "bddc_destroy", "bddc_setup", "bddc_refactor", "bddc_apply", "bddc_harmonic",
    "bddc_spmv", "bddc_pcg", "bddc_pcg_host", "bddc_solve_host", "bddc_get_stats", "bddc_sync",
    "bddc_kernel_launches_per_apply", "bddc_debug_copy", "bddc_launch_count",
    "bddc_event_record", "bddc_event_elapsed_ms", "bddc_profile", "bddc_profile_read",
    "bddc_nccl_unique_id", "bddc_nccl_selftest", "bddc_comm_init_nccl", "bddc_comm_init_host", "bddc_partition_info",
    "bddc_dense_potrf", "bddc_dense_trsm", "bddc_dense_gemm", "bddc_dense_gemv_t", "bddc_check", "bddc_update_weights",
    "bddc_coarse_solve", "bddc_set_coarse_solver", "bddc_coarse_elements", "bddc_read_buffer", "bddc_coarse_pattern",
    "bddc_index_build", "bddc_index_size", "bddc_index_copy", "bddc_index_free", "bddc_coarse_csr",
    "bddc_layout_tables", "bddc_nd_build", "bddc_nd_size", "bddc_nd_copy", "bddc_nd_free",
)


class SetupDesc(C.Structure):
    _fields_ = [
        ("dim", _i), ("cells", _i * 3), ("subs", _i * 3), ("element", _i), ("coarse_scaling", _i),
        ("alpha", _pd), ("elem_K", _pd),
        ("nloc_nodes", _i), ("nG", _i), ("nG_pad", _i), ("m", _i), ("m_pad", _i), ("nblk", _i),
        ("nI_pad", _i), ("nc_pad", _i),
        ("node_code", _pi), ("slot_node", _pi), ("irow_node", _pi),
        ("slot_gamma", _pi), ("slot_w", _pd), ("slot_con", _pi), ("slot_coef", _pd),
        ("con_coarse", _pi),
        ("n_gamma", _i), ("gamma_dof", _pll), ("gamma_slots", _pi),
        ("n_coarse", _i), ("coarse_slots", _pi),
        ("nnodes", _i), ("node_sep_start", _pi), ("node_sep_size", _pi), ("node_level", _pi),
        ("node_parent", _pi), ("bnd_ptr", _pi), ("bnd_idx", _pi), ("rmap", _pi),
        ("nnz", _ll), ("csr_node", _pi), ("csr_row", _pi), ("csr_col", _pi), ("seg_ptr", _pll),
        ("ncontrib", _ll), ("contrib", _pi),
    ]


class PcgReport(C.Structure):
    _fields_ = [("iterations", _i), ("converged", _i), ("bad_value", _d), ("bad_kind", _i)]


class Stats(C.Structure):
    _fields_ = [
        ("t_upload_ms", _d), ("t_local_ms", _d), ("t_coarse_ms", _d),
        ("n", _ll), ("n_gamma", _ll), ("n_coarse", _ll), ("nsub", _ll),
        ("factor_bytes", _ll), ("front_bytes", _ll), ("workspace_bytes", _ll),
        ("nG_pad", _i), ("nI_pad", _i), ("m_pad", _i), ("nblk", _i), ("nc_pad", _i),
        ("nlevels", _i), ("max_front", _i),
        ("t_in_coarse_factor", _i), ("tv_in_coarse_solve", _i),
    ]


_lib = None


def load(required: bool = True):
    """Load the library (no GPU needed to load); raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if required:
            raise RuntimeError(
                f"CUDA library {LIB_PATH} not built; run `make` or __graft_entry__.build() "
                "(there is no CPU fallback)")
        return None
    lib = C.CDLL(LIB_PATH)
    lib.bddc_create.argtypes = [_i, C.POINTER(_vp)]
    lib.bddc_destroy.argtypes = [_vp]
    lib.bddc_destroy.restype = None
    lib.bddc_setup.argtypes = [_vp, C.POINTER(SetupDesc), C.c_char_p, C.c_size_t]
    lib.bddc_refactor.argtypes = [_vp, _pd, C.c_char_p, C.c_size_t]
    lib.bddc_apply.argtypes = [_vp, _vp, _vp, _vp]
    lib.bddc_harmonic.argtypes = [_vp, _vp, _vp, _vp]
    lib.bddc_spmv.argtypes = [_vp, _vp, _vp, _vp]
    lib.bddc_pcg.argtypes = [_vp, _vp, _vp, _d, _i, _pd, _pd, _pd, C.POINTER(PcgReport),
                             C.c_char_p, C.c_size_t]
    lib.bddc_pcg_host.argtypes = [_vp, _pd, _pd, _d, _i, _pd, _pd, _pd, C.POINTER(PcgReport),
                                  C.c_char_p, C.c_size_t]
    lib.bddc_solve_host.argtypes = [_vp, _pd, _pd, _pd, _d, _i, _pd, _pd, _pd, C.POINTER(PcgReport),
                                    C.c_char_p, C.c_size_t]
    lib.bddc_get_stats.argtypes = [_vp, C.POINTER(Stats)]
    lib.bddc_sync.argtypes = [_vp]
    lib.bddc_check.argtypes = [_vp, C.c_char_p, C.c_size_t]
    lib.bddc_update_weights.argtypes = [_vp, _pd, C.c_char_p, C.c_size_t]
    lib.bddc_coarse_solve.argtypes = [_vp, _vp, _vp, _vp]
    lib.bddc_set_coarse_solver.argtypes = [_vp, COARSE_SOLVER_FN, _vp]
    lib.bddc_coarse_elements.argtypes = [_vp, _pll]
    lib.bddc_coarse_elements.restype = C.c_void_p
    lib.bddc_kernel_launches_per_apply.argtypes = [_vp]
    lib.bddc_debug_copy.argtypes = [_vp, C.c_char_p, _pd, _ll]
    lib.bddc_debug_copy.restype = _ll
    lib.bddc_read_buffer.argtypes = [_vp, C.c_char_p, _ll, _ll, _pd]
    lib.bddc_read_buffer.restype = _ll
    lib.bddc_coarse_pattern.argtypes = [_i, _pll, _pll, _pll, _ll, _i, _i, _pll, _pll, _pll, _pll, _pll, _pll,
                                        _pll, _pll, _pll, _pll, _pi]
    lib.bddc_coarse_pattern.restype = _ll
    lib.bddc_index_build.argtypes = [_i, _i, _pi, _pi, _pi, _i, C.POINTER(_vp), C.c_char_p, C.c_size_t]
    lib.bddc_index_size.argtypes = [_vp, C.c_char_p]
    lib.bddc_index_size.restype = _ll
    lib.bddc_index_copy.argtypes = [_vp, C.c_char_p, _vp, _ll]
    lib.bddc_index_free.argtypes = [_vp]
    lib.bddc_index_free.restype = None
    lib.bddc_layout_tables.argtypes = [_i, _i, _pi, _pi, _i, _i, _i, _pi, _pi, _ll, _pi, _i, _pi, _pd, _pi, _i,
                                       _pi, _pd, _pll, _pi, _pi, _pi, _pd, _pd, _pi, C.c_char_p, C.c_size_t]
    lib.bddc_nd_build.argtypes = [_ll, _i, _pi, _i, _i, _pi, _pi, _pll, _pll, C.POINTER(_vp), C.c_char_p, C.c_size_t]
    lib.bddc_nd_size.argtypes = [_vp, C.c_char_p]
    lib.bddc_nd_size.restype = _ll
    lib.bddc_nd_copy.argtypes = [_vp, C.c_char_p, _pll, _ll]
    lib.bddc_nd_free.argtypes = [_vp]
    lib.bddc_nd_free.restype = None
    lib.bddc_coarse_csr.argtypes = [_vp, _pll, _pll, _pll, _pi, _ll, _ll]
    lib.bddc_coarse_csr.restype = _ll
    lib.bddc_launch_count.argtypes = []
    lib.bddc_launch_count.restype = _ll
    lib.bddc_event_record.argtypes = [_vp, _i]
    lib.bddc_event_elapsed_ms.argtypes = [_vp, _i, _i]
    lib.bddc_event_elapsed_ms.restype = _d
    lib.bddc_profile.argtypes = [_vp, _i]
    lib.bddc_profile_read.argtypes = [_vp, C.c_char_p, _pll]
    lib.bddc_profile_read.restype = _d
    lib.bddc_nccl_unique_id.argtypes = [_vp]
    lib.bddc_nccl_selftest.argtypes = [_i]
    lib.bddc_comm_init_nccl.argtypes = [_vp, _i, _i, _vp]
    lib.bddc_comm_init_host.argtypes = [_vp, _i, _i, _vp, _vp]
    lib.bddc_partition_info.argtypes = [_i, _pi, _pi, _i, _i, _pll]
    lib.bddc_dense_potrf.argtypes = [_vp, _i, _i, _ll, _i, _pi, _vp]
    lib.bddc_dense_trsm.argtypes = [_i, _vp, _i, _i, _ll, _vp, _i, _i, _ll, _i, _vp]
    lib.bddc_dense_gemm.argtypes = [_i, _i, _i, _i, _i, _d, _vp, _i, _ll, _vp, _i, _ll, _d, _vp,
                                    _i, _ll, _i, _vp]
    lib.bddc_dense_gemv_t.argtypes = [_i, _i, _d, _vp, _i, _ll, _vp, _ll, _d, _vp, _ll, _i, _vp]
    _lib = lib
    return lib


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))
