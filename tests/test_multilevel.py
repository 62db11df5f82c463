"""Three-level BDDC-SO (the paper's outlook; the reference has no such level, so
there is nothing to pin against): the level-2 preconditioner is checked through the properties
the method guarantees, on the level-1 coarse problems of the oracle (test infrastructure)."""
import os
import sys

import numpy as np
import pytest
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from oracle import bddc_oracle as O  # noqa: E402
from paper_2001_07289_b200.multilevel import Level2Bddc, box_of_subdomains  # noqa: E402


def _coarse_elements(orc):
    """(ids, mats) of the oracle's coarse problem: S_0i = Ψ_iᵀ A_i Ψ_i (bddc.py:494-505)."""
    ncp = max(L.m for L in orc.locals)
    ids = -np.ones((len(orc.locals), ncp), dtype=np.int64)
    mats = np.zeros((len(orc.locals), ncp, ncp))
    for i, L in enumerate(orc.locals):
        S = L.psi.T @ (L.A @ L.psi)
        ids[i, :L.m] = L.coarse_ids
        mats[i, :L.m, :L.m] = 0.5 * (S + S.T)
    return ids, mats


CASES = [
    dict(dim=2, cells=(32, 32), subs=(8, 8), split=2, k=2, element="p1", mode="spec"),
    dict(dim=2, cells=(32, 32), subs=(8, 8), split=1, k=4, element="q1", mode="reference"),
    dict(dim=3, cells=(16, 16, 16), subs=(4, 4, 4), split=2, k=2, element="p1", mode="reference"),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['dim']}d_{c['subs'][0]}_k{c['k']}_{c['mode']}")
def test_level2_is_spd_and_bounded(case):
    orc = O.Oracle(case["dim"], case["cells"], case["subs"], case["split"], element=case["element"],
                   coarse_scaling=case["mode"])
    ids, mats = _coarse_elements(orc)
    box = box_of_subdomains(case["subs"], case["k"])
    n0 = orc.n_coarse
    M = Level2Bddc(ids, torch.from_numpy(mats), box, n0, checker=True)
    assert M.n_boxes == np.prod([s // case["k"] for s in case["subs"]])
    assert M.n_coarse2 < n0 and M.n_gamma2 < n0
    B = M.dense().numpy()
    assert np.abs(B - B.T).max() <= 1e-10 * np.abs(B).max()
    S0 = orc.coarse.toarray()
    # element matrices assemble to the reference's coarse matrix
    A = np.zeros_like(S0)
    for e in range(len(ids)):
        v = ids[e][ids[e] >= 0]
        A[np.ix_(v, v)] += mats[e][: len(v), : len(v)]
    assert np.abs(A - S0).max() <= 1e-10 * np.abs(S0).max()
    lam = np.linalg.eigvals(0.5 * (B + B.T) @ S0).real
    assert lam.min() >= 1.0 - 1e-8          # BDDC: the preconditioned spectrum is bounded below by 1
    assert lam.max() / lam.min() <= 12.0    # and by C (1 + log(H/h))^2 above


def test_three_level_pcg_matches_two_level():
    """The level-1 apply with S_0⁻¹ replaced by the level-2 preconditioner is still an SPD
    preconditioner: PCG converges to the same solution in a few more iterations."""
    case = CASES[2]
    orc = O.Oracle(case["dim"], case["cells"], case["subs"], case["split"], element=case["element"],
                   coarse_scaling="spec")
    b = O.uniform_f(orc.mesh.n_free, 0)
    x2, rep2 = O.pcg(orc.matvec, orc.apply, b, tol=1e-8)
    ids, mats = _coarse_elements(orc)
    M = Level2Bddc(ids, torch.from_numpy(mats), box_of_subdomains(case["subs"], case["k"]), orc.n_coarse, checker=True)

    class Fac:
        def solve(self, r):
            return M.solve(torch.from_numpy(np.ascontiguousarray(r))).numpy()

    orc.coarse_fac = Fac()
    x3, rep3 = O.pcg(orc.matvec, orc.apply, b, tol=1e-8)
    it2 = rep2["iterations"] if isinstance(rep2, dict) else rep2.iterations
    it3 = rep3["iterations"] if isinstance(rep3, dict) else rep3.iterations
    assert it2 <= it3 <= it2 + 8
    assert np.linalg.norm(x3 - x2) <= 1e-6 * np.linalg.norm(x2)


def test_box_of_subdomains():
    b = box_of_subdomains((4, 2), 2)
    assert b.tolist() == [0, 0, 1, 1, 0, 0, 1, 1]
    b3 = box_of_subdomains((2, 2, 4), (2, 2, 2))
    assert b3.tolist() == [0] * 8 + [1] * 8


def test_stiffness_weights_are_a_partition_of_unity():
    case = CASES[0]
    orc = O.Oracle(case["dim"], case["cells"], case["subs"], case["split"], element=case["element"],
                   coarse_scaling=case["mode"])
    ids, mats = _coarse_elements(orc)
    M = Level2Bddc(ids, torch.from_numpy(mats), box_of_subdomains(case["subs"], case["k"]), orc.n_coarse,
                   weights="stiffness", checker=True)
    tot = torch.zeros(M.n0 + 1, dtype=torch.float64)
    tot.index_add_(0, M.idxG.reshape(-1), M.wG.reshape(-1))
    on_g2 = torch.unique(M.idxG[M.idxG < M.n0])
    assert float((tot[on_g2] - 1.0).abs().max()) <= 1e-12
    B = M.dense().numpy()
    assert np.abs(B - B.T).max() <= 1e-10 * np.abs(B).max()
    lam = np.linalg.eigvals(0.5 * (B + B.T) @ orc.coarse.toarray()).real
    assert lam.min() >= 1.0 - 1e-8
    with pytest.raises(ValueError):
        Level2Bddc(ids, torch.from_numpy(mats), box_of_subdomains(case["subs"], case["k"]), orc.n_coarse,
                   weights="nope", checker=True)


def test_level2_refuses_cpu_without_checker_flag():
    ids = np.array([[0, 1], [1, 2]])
    mats = np.tile(np.array([[1.0, -1.0], [-1.0, 1.0]]) + np.eye(2), (2, 1, 1))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        Level2Bddc(ids, torch.from_numpy(mats), np.array([0, 1]), 3)
