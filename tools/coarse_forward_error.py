"""Forward error of the device coarse solve on a full-size pin (default cfg4), estimated by one
step of iterative refinement with the residual accumulated in extended precision on the host:
y1 = S0^-1 q (device factor), rho = q - S0 y1 (np.longdouble), dy = S0^-1 rho; |dy| / |y1| is the
relative forward error of y1 up to second order. Also SuperLU (the reference's coarse solver,
linalg.py:117-138) on the same matrix and right-hand side, refined the same way, and the
difference of the two solutions. Usage: python tools/coarse_forward_error.py [case]"""
import os
import sys

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import paper_2001_07289_b200 as P  # noqa: E402
from conftest import GOLDEN, Golden, build_problem  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
with np.load(os.path.join(GOLDEN, "fullsize", case + ".npz")) as f:
    g = Golden({k: f[k] for k in f.files})
pb = build_problem(g, device=0)
op = P.build_bddc(pb["system"], pb["pair"], pb["objects"], pb["recipe"], pb["weights"], coarse_scaling=pb["mode"])
S = op.coarse_matrix  # SparseSym (upper triangle stored)
A = S.tocsr()  # both triangles
n = A.shape[0]
d = A.diagonal()
print(f"{case}: coarse n = {n}, diag range {d.min():.3e} .. {d.max():.3e}")
q = np.random.default_rng(7).standard_normal(n) * np.sqrt(d)  # rhs scaled like the matrix rows


def resid_ld(y):
    Al = A.astype(np.longdouble)
    return (q.astype(np.longdouble) - Al @ y.astype(np.longdouble)).astype(np.float64)


def refine(solve, name):
    y1 = solve(q)
    rho = resid_ld(y1)
    dy = solve(rho)
    print(f"{name}: residual |q - S0 y| / |q| = {np.linalg.norm(rho) / np.linalg.norm(q):.3e}, "
          f"forward error |dy| / |y| = {np.linalg.norm(dy) / np.linalg.norm(y1):.3e} "
          f"(max-norm {np.abs(dy).max() / np.abs(y1).max():.3e})")
    return y1, y1 + dy


y_dev, y_dev2 = refine(op.coarse_factor.solve, "device multifrontal")
lu = spla.splu(A.tocsc())
y_lu, y_lu2 = refine(lu.solve, "SuperLU (reference solver)")
print(f"device vs SuperLU: |y_dev - y_lu| / |y| = {np.linalg.norm(y_dev - y_lu) / np.linalg.norm(y_lu):.3e}; "
      f"after refinement {np.linalg.norm(y_dev2 - y_lu2) / np.linalg.norm(y_lu2):.3e}")
print(f"device error vs refined SuperLU {np.linalg.norm(y_dev - y_lu2) / np.linalg.norm(y_lu2):.3e}; "
      f"SuperLU error vs refined device {np.linalg.norm(y_lu - y_dev2) / np.linalg.norm(y_dev2):.3e}")
