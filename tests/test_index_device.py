"""Device index sets (csrc/index_sets.cu) against the reference fixtures and
the host statement: membership / Γ (partition.py:117-131, 75-83), objects
(partition.py:223-250), counting / cardinality weights (bddc.py:108-145). Bit-exact."""
import numpy as np
import pytest

import paper_2001_07289_b200 as P
from conftest import build_problem, golden_cases, load_golden

pytestmark = pytest.mark.gpu


def _same_objects(a, b):
    for f in ("signature", "sig_len", "owners", "owner_len", "kind", "dof_ptr", "dof_list", "dof_obj"):
        x, y = getattr(a, f), getattr(b, f)
        assert x.dtype == y.dtype and np.array_equal(x, y), f


@pytest.mark.parametrize("case", golden_cases())
def test_device_index_sets_match_reference_fixtures(cuda_ok, case):
    g = load_golden(case)
    pb = build_problem(g, device=0)
    pair, objs, w = pb["pair"], pb["objects"], pb["weights"]
    assert hasattr(objs, "_device_weights")
    cons = P.select_constraints(objs, pb["recipe"], pair)
    assert np.array_equal(pair.membership.gamma_dofs, g["gamma_dofs"])
    assert np.array_equal(objs.signature, g["obj_sig"])
    assert np.array_equal(objs.owners, g["obj_owners"])
    assert np.array_equal(objs.kind, g["obj_kind"])
    assert np.array_equal(objs.dof_ptr, g["obj_dof_ptr"])
    assert np.array_equal(objs.dof_list, g["obj_dofs"])
    assert np.array_equal(cons.con_obj, g["con_obj"])
    assert np.array_equal(cons.dof_list, g["con_dofs"])
    assert np.array_equal(cons.coeff, g["con_coeff"])
    assert len(cons) == int(g["coarse_size"])
    assert np.array_equal(w.weights_for(g["w_sub"], g["w_dof"]), g["w_val"])


@pytest.mark.parametrize("dim,cells,subs,split,coef", [
    (2, (96, 64), (6, 4), 4, None),
    (2, (64, 64), (4, 4), 16, None),          # L = h: every interface dof a vertex
    (3, (48, 48, 48), (6, 6, 6), 2, None),
    (3, (32, 24, 16), (4, 3, 2), 1, None),    # Θ̂ = Θ
    (3, (24, 24, 24), (3, 3, 3), -1, 1),      # refine_by_coefficient on random blocks
    (2, (64, 64), (4, 4), -1, 2),
])
def test_device_matches_host_statement(cuda_ok, dim, cells, subs, split, coef):
    mesh = P.build_mesh(dim, cells, "p1")
    if coef is None:
        cf = P.make_constant(mesh, 1.0)
    else:  # blocks of 4 (3D) / 8 (2D) cells with two values: ragged, non-box Θ̂
        b = 4 if dim == 3 else 8
        multi = mesh.cell_multi_indices()
        nb = [c // b for c in cells]
        bid = sum((multi[:, d] // b) * int(np.prod(nb[:d])) for d in range(dim))
        vals = np.where(np.random.default_rng(coef).random(int(np.prod(nb))) < 0.5, 1.0, 100.0)
        cf = P.CoefficientField(vals[bid])
    theta = P.partition_uniform(mesh, subs)
    mk = (lambda: P.refine_by_coefficient(mesh, theta, cf, validate=False)) if split < 0 else (
        lambda: P.refine_uniform(mesh, theta, split, validate=False))
    ph, pd = mk(), mk()
    oh = P.classify_objects(ph)
    od = P.classify_objects(pd, device=0)
    assert np.array_equal(ph.membership.gamma_dofs, pd.membership.gamma_dofs)
    assert np.array_equal(ph.membership.gamma_hat_dofs, pd.membership.gamma_hat_dofs)
    _same_objects(oh, od)
    for mode in ("counting", "cardinality"):
        wh = P.compute_weights(ph, mode, cf, oh)
        wd = P.compute_weights(pd, mode, cf, od)
        assert np.array_equal(wh.obj_weights, wd.obj_weights), mode
    # the per-dof tuples are still available (materialised on the host on demand)
    d = int(pd.membership.gamma_dofs[0])
    assert pd.membership.on_gamma[d] == ph.membership.on_gamma[d]


def test_device_index_sets_at_cfg3_size(cuda_ok):
    """cfg3's index sets (128³, 16³ subdomains, split 2): device == host."""
    mesh = P.build_mesh(3, (128, 128, 128), "p1")
    theta = P.partition_uniform(mesh, (16, 16, 16))
    ph = P.refine_uniform(mesh, theta, 2, validate=False)
    pd = P.refine_uniform(mesh, theta, 2, validate=False)
    oh = P.classify_objects(ph)
    od = P.classify_objects(pd, device=0)
    _same_objects(oh, od)
    assert len(P.select_constraints(od, "vef", pd)) == P.count_coarse_dofs((16, 16, 16), 2, "vef") == 139455


@pytest.mark.parametrize("case", golden_cases())
def test_device_layout_tables_match_host(cuda_ok, case):
    """Per-subdomain slot tables (interface position, local constraint, coefficient, weight)
    and the interface gather table from the device kernels (bddc_layout_tables) equal the
    numpy statement (layout.py; bddc.py:420-490)."""
    from paper_2001_07289_b200.layout import build_device_plan

    g = load_golden(case)
    pb = build_problem(g)
    if pb["pair"].box_layout is None:
        pytest.skip("non-box partition")
    cons = P.select_constraints(pb["objects"], pb["recipe"], pb["pair"])
    h = build_device_plan(pb["pair"], cons, pb["weights"], coarse_pattern="device")
    d = build_device_plan(pb["pair"], cons, pb["weights"], coarse_pattern="device", device=0)
    for f in ("slot_gamma", "slot_con", "slot_coef", "slot_w", "gamma_slots", "con_coarse", "coarse_slots",
              "gamma_dof", "n_con_local"):
        a, b = getattr(h, f), getattr(d, f)
        assert a.dtype == b.dtype and np.array_equal(a, b), f
