"""Why the cfg4 analogue in the reference's coarse scaling cannot meet ±1 iterations: the
reference algorithm itself (the oracle, bit-identical to the reference on the unperturbed
input: tests/test_oracle_golden.py) changes its PCG iteration count by tens of iterations
when the right-hand side is perturbed at the level of its own rounding (relative 1e-16 ..
1e-14), while κ and x stay put. κ ≈ 8e8 makes the iteration count of this Krylov run
chaotic; the GPU path is held to the reference's own spread instead (test_gpu_scale.py)."""
import numpy as np

from conftest import load_golden
from oracle import bddc_oracle as orc


def test_reference_mode_cfg4_iterations_are_chaotic():
    g = load_golden("cfg4a_p1_ref")
    dim = int(g["dim"])
    cells = tuple(int(c) for c in g["cells"])
    subs = tuple(int(s) for s in g["subs"])
    o = orc.Oracle(dim, cells, subs, int(g["split"]), str(g["recipe"]), str(g["weighting"]), "p1",
                   orc.block_alpha(cells, 4, 0), "reference")
    b = np.asarray(g["b"], float)
    rng = np.random.default_rng(7)
    its = []
    for eps in (0.0, 1e-16, 1e-15, 1e-14):
        bb = b * (1 + eps * rng.standard_normal(len(b))) if eps else b
        x, rep = orc.pcg(o.matvec, o.apply, bb, float(g["tol"]), 2000)
        its.append(rep["iterations"])
        assert rep["converged"]
        assert abs(rep["kappa"] - float(g["kappa"])) <= 1e-6 * float(g["kappa"])
        assert np.linalg.norm(x - g["x"]) <= 1e-10 * np.linalg.norm(g["x"])
    assert its[0] == int(g["iterations"])      # unperturbed: the reference's count (1397)
    assert max(its) - min(its) > 2             # rounding-level noise moves it by far more than ±1
