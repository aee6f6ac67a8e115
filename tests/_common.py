"""Shared helpers: golden fixtures, seeded inputs, tolerances."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")
REF_SRC = "/root/reference/pkg/src"

# north star: relative L2 <= 1e-12 in fp64
RTOL = 1e-12

_gold = None


def golden():
    global _gold
    if _gold is None:
        _gold = dict(np.load(GOLDEN))
    return _gold


def inputs(n, seed=0):
    """b ~ U[-1,1](seed), x0 ~ U[-1,1](seed+1)."""
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, n)
    x0 = np.random.default_rng(seed + 1).uniform(-1.0, 1.0, n)
    return x0, b


def rel(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def have_reference():
    return os.path.isdir(REF_SRC)


GOLDEN_MG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_mg.npz")
_gold_mg = None


def golden_mg():
    global _gold_mg
    if _gold_mg is None:
        _gold_mg = dict(np.load(GOLDEN_MG))
    return _gold_mg


def useed(n, seed):
    """default_rng(seed).uniform(-1, 1, n) (tests/golden/make_golden_mg.py)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def rhs_f(x):
    """Source term of the compute_rhs fixtures (tests/golden/make_golden_mg.py)."""
    return np.sin(np.pi * x[:, 0]) * np.cos(0.5 * np.pi * x[:, -1]) + 0.25 * x.sum(axis=1)


def rhs_g(x):
    """Dirichlet data of the compute_rhs fixtures."""
    return x[:, 0] ** 2 - 0.5 * x[:, -1] + 0.125


REF_INSTALLED = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                             "baseline", "_ref")


def ref_dgmg():
    """The unmodified reference package `dgmg`: the copy `build()` installs
    into baseline/_ref (it travels to the GPU box), else the source tree in
    this container; None when neither exists.  Tests only (the checker)."""
    import importlib
    import sys
    for path in (REF_INSTALLED, REF_SRC):
        if os.path.isdir(os.path.join(path, "dgmg")):
            if path not in sys.path:
                sys.path.insert(0, path)
            return importlib.import_module("dgmg")
    return None


GOLDEN_BIG = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_big.npz")
_gold_big = None


def golden_big():
    """Degree 8..15 vertex-patch steps and 1D levels (tests/golden/make_golden_big.py)."""
    global _gold_big
    if _gold_big is None:
        _gold_big = dict(np.load(GOLDEN_BIG))
    return _gold_big
