"""The checked build (make check: libbddcso_b200_check.so, -DBDDC_CHECKS) on the parity cases:
every index-driven gather / scatter of the extend-add, the coarse assembly, the interface
gather and the coarse solve is bounds-checked on the device (a failure traps the launch).
compute-sanitizer is closed on this GPU pool; this is the bounds evidence instead. Each case
runs in a subprocess (the library is chosen at import) with aliased fronts and the L21 coarse
solve path forced on, and must still match the reference fixture."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK_LIB = os.path.join(ROOT, "paper_2001_07289_b200", "libbddcso_b200_check.so")

SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import paper_2001_07289_b200 as P
from paper_2001_07289_b200 import _capi
from conftest import build_problem, load_golden
assert _capi.LIB_PATH.endswith("libbddcso_b200_check.so")
g = load_golden({case!r})
pb = build_problem(g, device=0)
op = P.build_bddc(pb["system"], pb["pair"], pb["objects"], pb["recipe"], pb["weights"], coarse_scaling=pb["mode"])
z = op.apply(g["r"])
tol = 1e-9 if "cfg4" in {case!r} or "chan" in {case!r} else 1e-12
assert np.abs(z - g["Br"]).max() <= tol * np.abs(g["Br"]).max()
x, rep = P.pcg(op.matvec, op.apply, g["b"], tol=float(g["tol"]), max_iters=2000)
assert abs(rep.iterations - int(g["iterations"])) <= 1
op.refactor()
op.close()
print("checked ok")
"""


@pytest.mark.parametrize("case", ["cfg1_p1_ref", "cfg2a_p1_L4h", "cfg3a_p1_ref", "cfg3c_p1_ref", "cfg4a_p1_spec",
                                  "chan_q1_coeff"])
def test_checked_build_parity(cuda_ok, case):
    if not os.path.exists(CHECK_LIB):
        pytest.fail("checked library missing: run `make check` (built by __graft_entry__.build())")
    env = dict(os.environ, BDDC_LIB=CHECK_LIB, BDDC_FRONT_ALIAS="1", BDDC_FRONT_ALIAS_MIN_MB="0",
               BDDC_W21_MAX_SEP="128")
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), case=case)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "checked ok" in r.stdout, (r.stdout[-2000:], r.stderr[-4000:])
    assert "BDDC_CHECK failed" not in r.stdout + r.stderr
