"""CPU check of the device formulation (Schur complement + augmented Lagrangian local
solves, nested-dissection multifrontal coarse solve) over the same host tables the GPU
uses, against the reference fixtures."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import build_problem, load_golden
from device_emulator import Emulator
from oracle import bddc_oracle as orc
from paper_2001_07289_b200 import select_constraints
from paper_2001_07289_b200.layout import build_device_plan

CASES = ["cfg1_p1_ref", "cfg1_p1_spec", "cfg1_q1_ref", "cfg2a_p1_Lh", "cfg3a_p1_ref",
         "cfg4a_p1_spec", "full_p1_2d", "q1_3d_vf"]


@pytest.mark.parametrize("case", CASES)
def test_emulated_device_algorithm(case):
    g = load_golden(case)
    pb = build_problem(g)
    cons = select_constraints(pb["objects"], pb["recipe"], pb["pair"])
    plan = build_device_plan(pb["pair"], cons, pb["weights"])
    em = Emulator(pb["system"], pb["pair"], plan, pb["mode"])
    tol_apply = 1e-9 if "cfg4" in case else 1e-12
    Br = em.apply(g["r"])
    assert np.abs(Br - g["Br"]).max() <= tol_apply * np.abs(g["Br"]).max()
    n = len(cons)
    ref = sp.csr_matrix((g["coarse_data"], g["coarse_indices"], g["coarse_indptr"]), shape=(n, n)).toarray()
    mine = em.S0_elim[np.ix_(plan.coarse.iperm, plan.coarse.iperm)]
    assert np.abs(mine - ref).max() <= 1e-13 * np.abs(ref).max()
    x, rep = orc.pcg(em.A.dot, em.apply, g["b"], float(g["tol"]))
    assert abs(rep["iterations"] - int(g["iterations"])) <= 1
    assert abs(rep["kappa"] - float(g["kappa"])) <= 1e-6 * float(g["kappa"])
    assert np.linalg.norm(x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])
