"""Host index sets (partition, membership, objects, weights, constraints): bit-exact
against fixtures generated from the reference; SPEC known-answer tests."""
import numpy as np
import pytest

import paper_2001_07289_b200 as P
from conftest import build_problem, golden_cases, load_golden


@pytest.mark.parametrize("case", golden_cases())
def test_index_sets_bit_exact(case):
    g = load_golden(case)
    pb = build_problem(g)
    pair, objs, w = pb["pair"], pb["objects"], pb["weights"]
    cons = P.select_constraints(objs, pb["recipe"], pair)
    if "theta_hat" in g:  # refine_by_coefficient labels (partition.py:202-220)
        assert np.array_equal(pair.theta_hat, g["theta_hat"])
        assert np.array_equal(pb["coeff"].alpha, g["alpha"])
    assert np.array_equal(pair.membership.gamma_dofs, g["gamma_dofs"])
    assert np.array_equal(objs.signature, g["obj_sig"])
    assert np.array_equal(objs.owners, g["obj_owners"])
    assert np.array_equal(objs.kind, g["obj_kind"])
    assert np.array_equal(objs.dof_ptr, g["obj_dof_ptr"])
    assert np.array_equal(objs.dof_list, g["obj_dofs"])
    assert np.array_equal(cons.con_obj, g["con_obj"])
    assert np.array_equal(cons.dof_ptr, g["con_ptr"])
    assert np.array_equal(cons.dof_list, g["con_dofs"])
    assert np.array_equal(cons.coeff, g["con_coeff"])
    assert len(cons) == int(g["coarse_size"])
    # weights are bit-exact (exact rationals rounded once)
    assert np.array_equal(w.weights_for(g["w_sub"], g["w_dof"]), g["w_val"])


def test_count_coarse_dofs_kat():
    g = load_golden("count_kat")
    for s in (1, 2, 4, 6, 8):
        assert P.count_coarse_dofs((10, 10, 10), s, "vef") == int(g[str(s)])
    # SPEC.md:167-169 / PAPER Table 1
    assert [P.count_coarse_dofs((10, 10, 10), s, "vef") for s in (1, 2, 4, 6)] == [5859, 32319, 150039, 354159]


def test_object_table_behaves_like_list():
    mesh = P.build_mesh(2, (8, 8), "p1")
    pair = P.refine_uniform(mesh, P.partition_uniform(mesh, (2, 2)), 2)
    objs = P.classify_objects(pair)
    assert len(list(objs)) == len(objs)
    o = objs[0]
    assert o.id == 0 and o.kind in ("vertex", "edge") and len(o.signature) >= 2
    assert objs[-1].id == len(objs) - 1
    ms = pair.membership
    assert isinstance(ms.on_gamma[int(ms.gamma_dofs[0])], tuple)


def test_spec_fig1_weights():
    """SPEC.md:297 / PAPER Fig. 1: δ†(ξ) = 2/3 cardinality vs 1/2 counting at a point shared
    by 3 subsubdomains of which 2 belong to one subdomain."""
    from fractions import Fraction

    mesh = P.build_mesh(2, (4, 4), "q1")
    theta = P.partition_uniform(mesh, (2, 1))           # left / right halves
    theta_hat = theta.copy() * 2
    multi = mesh.cell_multi_indices()
    theta_hat[(theta == 0) & (multi[:, 1] >= 2)] = 1    # left half split top / bottom
    theta_hat[theta == 1] = 2
    pair = P.PartitionPair(mesh, theta, theta_hat)
    w_card = P.compute_weights(pair, "cardinality")
    w_cnt = P.compute_weights(pair, "counting")
    # dof at node (2, 2): cells of hats {0, 1, 2}; subdomain 0 owns 2 of the 3
    dof = int(mesh.node_to_free[2 + 5 * 2])
    assert w_card.weight_fraction(0, dof) == Fraction(2, 3)
    assert w_card.weight(1, dof) == float(Fraction(1, 3))
    assert w_cnt.weight(0, dof) == 0.5


def test_recipe_errors():
    mesh = P.build_mesh(3, (8, 8, 8), "q1")
    pair = P.refine_uniform(mesh, P.partition_uniform(mesh, (4, 4, 4)), 1)
    objs = P.classify_objects(pair)
    with pytest.raises(P.RecipeError):
        P.select_constraints(objs, "f", pair)  # faces only: floating interior subdomain paths
    cons = P.select_constraints(objs, "vef", pair)
    assert len(cons) == P.count_coarse_dofs((4, 4, 4), 1, "vef")


def test_partition_validation_errors():
    mesh = P.build_mesh(2, (4, 4))
    theta = np.zeros(16, dtype=np.int64)
    theta[[0, 15]] = 1  # two corner cells: disconnected part 1
    with pytest.raises(ValueError, match="not face-connected"):
        P.PartitionPair(mesh, theta, theta)
    with pytest.raises(ValueError, match="spans subdomains"):
        P.PartitionPair(mesh, P.partition_uniform(mesh, (2, 2)), np.zeros(16, dtype=np.int64))


def test_refine_by_coefficient_matches_uniform_cells():
    mesh = P.build_mesh(3, (16, 16, 16), "p1")
    cf = P.make_blocks(mesh, 4, 0)
    theta = P.partition_uniform(mesh, (2, 2, 2))
    a = P.refine_by_coefficient(mesh, theta, cf)
    b = P.refine_uniform(mesh, theta, 2)
    # same cell groups (different labels), SURVEY §8 cfg4 row
    pairs = np.unique(np.stack([a.theta_hat, b.theta_hat], axis=1), axis=0)
    assert len(pairs) == a.subsubdomain_count == b.subsubdomain_count


def test_refine_by_coefficient_matches_reference_labels():
    g = load_golden("refine_coeff")
    mesh = P.build_mesh(3, tuple(int(c) for c in g["cells"]), "q1")
    cf = P.CoefficientField(g["alpha"])
    pair = P.refine_by_coefficient(mesh, P.partition_uniform(mesh, tuple(int(s) for s in g["subs"])), cf)
    assert np.array_equal(pair.theta_hat, g["theta_hat"])
