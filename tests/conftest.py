import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

GOLDEN = os.path.join(ROOT, "tests", "golden")
CHANNELS = {2: (3.0, 2, 2, 0), 3: (3.0, 2, 2, 1)}  # as oracle/make_golden.py


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and the built library")


def golden_cases(big=None):
    """Fixture names; big=False: the small cases (oracle-pinned), True: the scale cases
    (reference run without partition validation, oracle/make_golden.py BIG_CASES)."""
    names = sorted(f[:-4] for f in os.listdir(GOLDEN)
                   if f.endswith(".npz") and f not in ("count_kat.npz", "refine_coeff.npz"))
    if big is None:
        return names
    return [n for n in names if is_big(n) == big]


def is_big(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as g:
        return "big" in g.files


def is_uniform(name):
    """Θ̂ from refine_uniform (the oracle's only refinement)."""
    with np.load(os.path.join(GOLDEN, name + ".npz")) as g:
        return "refine" not in g.files


class Golden(dict):
    """A fixture's arrays; ``r`` and ``b`` of the scale cases are regenerated from their seeds
    (r = default_rng(1234).standard_normal(n); b = h^d f with f ~ U[-1,1] seed 0, or the
    f = 1 load), exactly as oracle/make_golden.py drew them."""

    def __missing__(self, key):
        import paper_2001_07289_b200 as P

        if key == "r":
            v = np.random.default_rng(1234).standard_normal(int(self["n"]))
        elif key == "b":
            mesh = P.build_mesh(int(self["dim"]), tuple(int(c) for c in self["cells"]), str(self["element"]))
            f = P.uniform_source(mesh, 0) if str(self["rhs_kind"]) == "uniform" else 1.0
            v = P.mesh.load_vector(mesh, f)
        else:
            raise KeyError(key)
        self[key] = v
        return v


def load_golden(name):
    with np.load(os.path.join(GOLDEN, name + ".npz")) as g:
        return Golden({k: g[k] for k in g.files})


def build_problem(g, device=None):
    """Host problem (mesh, pair, objects, weights, constraints, system, rhs) of a fixture;
    ``device``: membership / objects / weights from the device index-set kernels."""
    import paper_2001_07289_b200 as P

    dim = int(g["dim"])
    cells = tuple(int(c) for c in g["cells"])
    subs = tuple(int(s) for s in g["subs"])
    mesh = P.build_mesh(dim, cells, str(g["element"]))
    kind = str(g["coeff"])
    if kind == "blocks":
        cf = P.make_blocks(mesh, 4, 0)
    elif kind == "channels":
        cf = P.make_channels(mesh, subs, P.ChannelSpec(*CHANNELS[dim]))
    else:
        cf = P.make_constant(mesh, 1.0)
    theta = P.partition_uniform(mesh, subs)
    if int(g["split"]) < 0:
        pair = P.refine_by_coefficient(mesh, theta, cf)
    else:
        pair = P.refine_uniform(mesh, theta, int(g["split"]), validate=False)
    objs = P.classify_objects(pair, device=device)
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
