import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built library")


def golden_cases():
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f not in ("count_kat.npz", "refine_coeff.npz"))


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def build_problem(g):
    """Host problem (mesh, pair, objects, weights, constraints, system, rhs) of a fixture."""
    import paper_2001_07289_b200 as P

    dim = int(g["dim"])
    cells = tuple(int(c) for c in g["cells"])
    subs = tuple(int(s) for s in g["subs"])
    mesh = P.build_mesh(dim, cells, str(g["element"]))
    cf = P.make_blocks(mesh, 4, 0) if str(g["coeff"]) == "blocks" else P.make_constant(mesh, 1.0)
    pair = P.refine_uniform(mesh, P.partition_uniform(mesh, subs), int(g["split"]))
    objs = P.classify_objects(pair)
    w = P.compute_weights(pair, str(g["weighting"]), cf, objs)
    recipe = P.Recipe.full() if bool(g["full"]) else str(g["recipe"])
    system = P.assemble(mesh, cf)
    return dict(mesh=mesh, coeff=cf, pair=pair, objects=objs, weights=w, recipe=recipe,
                system=system, mode=str(g["mode"]))


@pytest.fixture(scope="session")
def cuda_ok():
    try:
        import torch
    except Exception:
        pytest.skip("torch missing")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
