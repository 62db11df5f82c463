"""Native host symbolic work (csrc/host_plan.cu) against its numpy statement (symbolic.py):
bit-exact coarse CSR pattern, contribution lists and front positions. No GPU needed."""
import numpy as np
import pytest

import paper_2001_07289_b200 as P
from paper_2001_07289_b200 import layout, symbolic
from conftest import build_problem, load_golden


@pytest.mark.parametrize("case", ["cfg1_p1_ref", "cfg2a_p1_Lh", "cfg3b_p1_ref", "q1_3d_vf", "chan_q1_coeff",
                                  "cfg2b_p1_Lh44"])
def test_coarse_pattern_native_matches_numpy(case, monkeypatch):
    g = load_golden(case)
    pb = build_problem(g)
    cons = P.select_constraints(pb["objects"], pb["recipe"], pb["pair"])
    plans = {}
    for impl in ("numpy", "native"):
        monkeypatch.setattr(layout, "COARSE_CSR", symbolic.coarse_csr if impl == "numpy" else symbolic.coarse_csr_native)
        plans[impl] = layout.build_device_plan(pb["pair"], cons, pb["weights"]).coarse
    a, b = plans["numpy"], plans["native"]
    for k in ("csr_row", "csr_col", "csr_node", "csr_frow", "csr_fcol", "seg_ptr", "contrib"):
        assert np.array_equal(getattr(a, k), getattr(b, k)), k


@pytest.mark.parametrize("case", ["cfg1_p1_ref", "cfg2a_p1_Lh", "cfg2a_p1_L4h", "cfg3b_p1_ref", "q1_3d_vf",
                                  "chan_q1_coeff", "cfg2b_p1_Lh44", "cfg3c_p1_ref", "full_p1_2d"])
def test_nd_analysis_native_matches_numpy(case, monkeypatch):
    """bddc_nd_build (host_plan.cu) == symbolic.analyze: tree, elimination order, boundaries,
    extend-add maps."""
    g = load_golden(case)
    pb = build_problem(g)
    cons = P.select_constraints(pb["objects"], pb["recipe"], pb["pair"])
    plans = {}
    for impl in ("numpy", "native"):
        monkeypatch.setattr(layout, "ANALYZE", symbolic.analyze if impl == "numpy" else symbolic.analyze_native)
        plans[impl] = layout.build_device_plan(pb["pair"], cons, pb["weights"], coarse_pattern="device").coarse
    a, b = plans["numpy"], plans["native"]
    if a is None:
        assert b is None
        return
    for k in ("perm", "iperm", "sep_start", "sep_size", "level", "parent", "bnd_ptr", "bnd_idx", "rmap"):
        x, y = getattr(a, k), getattr(b, k)
        assert x.dtype == y.dtype and np.array_equal(x, y), k
