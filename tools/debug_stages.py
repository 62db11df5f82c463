"""Compare device intermediates with the numpy emulator (diagnostics)."""
import os, sys
import numpy as np
os.environ["BDDC_DEBUG_KEEP"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import paper_2001_07289_b200 as P
from conftest import build_problem, load_golden
from device_emulator import Emulator
case = sys.argv[1] if len(sys.argv) > 1 else "cfg1_p1_ref"
g = load_golden(case)
pb = build_problem(g)
op = P.build_bddc(pb["system"], pb["pair"], pb["objects"], pb["recipe"], pb["weights"], coarse_scaling=pb["mode"])
print("setup code", op.setup_code)
plan = op.plan
em = Emulator(pb["system"], pb["pair"], plan, pb["mode"])
lay = plan.layout
nsub, nG, ncp = plan.nsub, lay.nG_pad, plan.nc_pad
ds = op.debug_buffer("diag_s"); print("diag_s", ds[:4])
LS = op.debug_buffer("LS").reshape(nsub, nG, nG).transpose(0, 2, 1)
Phi = op.debug_buffer("Phi").reshape(nsub, ncp, nG).transpose(0, 2, 1)
Sl = op.debug_buffer("Sloc").reshape(nsub, ncp, ncp).transpose(0, 2, 1)
cs = op.debug_buffer("cscale")
for p in range(min(nsub, 4)):
    L = em.loc[p]
    nGr = lay.nG
    nc = int(plan.n_con_local[p])
    eLS = np.abs(np.tril(LS[p, :nGr, :nGr]) - L["LS"]).max() / np.abs(L["LS"]).max()
    ePhi = np.abs(Phi[p, :nGr, :nc] - L["Phi"]).max() / max(np.abs(L["Phi"]).max(), 1e-300)
    print(f"sub {p}: c {cs[p]:.6e} vs {L['c']:.6e}  LS {eLS:.2e}  Phi {ePhi:.2e}  Sloc00 {Sl[p,0,0]:.6e}")
cv = op.debug_buffer("csr_val")
cp = plan.coarse
ref = em.S0_elim[cp.csr_row, cp.csr_col]
print("csr_val err", np.abs(cv - ref).max() / np.abs(ref).max())
def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)
if op.setup_code == 0:
    z = op.apply(g["r"])
    ze = em.apply(g["r"])
    print("apply err", rel(z, g["Br"]), "emu err", rel(ze, g["Br"]))
    d = em.dbg
    print("u1", rel(op.debug_buffer("v1"), d["u1"]))
    gam = op.gamma_dofs
    print("rp_gamma", rel(op.debug_buffer("rpg"), d["rp"][gam]))
    U = op.debug_buffer("uloc").reshape(nsub, nG)
    T = op.debug_buffer("tloc").reshape(nsub, ncp)
    for p in range(min(nsub, 3)):
        u, t = d["st"][p]
        print(f" sub {p}: u {rel(U[p, :lay.nG], u):.2e} t {rel(T[p, :len(t)], t) if len(t) else 0:.2e}")
    cr = op.debug_buffer("crhs"); cs = op.debug_buffer("csol")
    print("crhs", rel(cr, d["crhs"]), "csol", rel(cs, d["csol"]))
    print("z", z[:5], "ze", ze[:5])
