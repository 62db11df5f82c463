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
