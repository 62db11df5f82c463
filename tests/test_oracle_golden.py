"""The CPU oracle (oracle/bddc_oracle.py) against fixtures generated from the reference.

Pins the oracle: identical iteration counts, B·r and x to round-off, κ to 1e-12.
"""
import numpy as np
import pytest

from conftest import golden_cases, is_uniform, load_golden
from oracle import bddc_oracle as orc

FAST = [c for c in golden_cases(big=False) if c != "cfg4a_p1_ref" and is_uniform(c)]


def _oracle(g):
    cells = tuple(int(c) for c in g["cells"])
    alpha = orc.block_alpha(cells, 4, 0) if str(g["coeff"]) == "blocks" else None
    return orc.Oracle(int(g["dim"]), cells, tuple(int(s) for s in g["subs"]), int(g["split"]),
                      str(g["recipe"]), str(g["weighting"]), str(g["element"]), alpha,
                      str(g["mode"]), bool(g["full"]))


@pytest.mark.parametrize("case", FAST)
def test_oracle_matches_reference(case):
    g = load_golden(case)
    o = _oracle(g)
    assert o.n_coarse == int(g["coarse_size"])
    Br = o.apply(g["r"])
    assert np.abs(Br - g["Br"]).max() <= 1e-13 * np.abs(g["Br"]).max()
    x, rep = orc.pcg(o.matvec, o.apply, g["b"], float(g["tol"]))
    assert rep["iterations"] == int(g["iterations"])
    assert abs(rep["kappa"] - float(g["kappa"])) <= 1e-12 * float(g["kappa"])
    assert np.linalg.norm(x - g["x"]) <= 1e-13 * np.linalg.norm(g["x"])


def test_oracle_p1_element_matches_product():
    from paper_2001_07289_b200.mesh import p1_kuhn_element_box, q1_element_box

    for h in ((0.25, 0.25), (1 / 64, 1 / 64), (0.125, 0.125, 0.125), (0.1, 0.2, 0.3)):
        assert np.array_equal(orc.p1_kuhn_element(list(h)), p1_kuhn_element_box(h))
        assert np.array_equal(orc.q1_element(list(h)), q1_element_box(h))


def test_source_generators_match():
    import paper_2001_07289_b200 as P

    mesh = P.build_mesh(2, (16, 16), "p1")
    assert np.array_equal(P.uniform_source(mesh, 3), orc.uniform_f(mesh.free_count, 3))
    m3 = P.build_mesh(3, (8, 8, 8), "p1")
    assert np.array_equal(P.make_blocks(m3, 4, 0).alpha, orc.block_alpha((8, 8, 8), 4, 0))
