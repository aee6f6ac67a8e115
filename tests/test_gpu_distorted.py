"""Distorted (multilinear) meshes: the device SIPG
operator against the reference's own `apply_operator` on the reference's
criterion-1 meshes (`test_acceptance.py:33-59`: distortion 0.25, seed 2024,
gamma_hat 4) and larger ones (tests/golden/make_golden_dist.py)."""
import os

import numpy as np
import pytest
import torch

from _common import rel, RTOL

from paper_1910_11239_b200 import distorted as D, mesh
from paper_1910_11239_b200.basis import Basis1D

pytestmark = pytest.mark.gpu
G = dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                              "golden_dist.npz")))
CASES = sorted({k.split("/")[0] for k in G})


def _ctx(name):
    d, coarse, level, k = (int(v) for v in G[name + "/meta"])
    h = D.distort(mesh.build_hierarchy(d, coarse, level), 0.25, 2024)
    return D.DistortedContext(h.levels[level], Basis1D.make(k), 4.0), h.levels[level]


@pytest.mark.parametrize("name", CASES)
def test_distorted_operator_matches_reference(name):
    ctx, lvl = _ctx(name)
    assert np.array_equal(lvl.vertex_grid, G[name + "/grid"])
    u = np.random.default_rng(3).uniform(-1.0, 1.0, ctx.ndofs)
    got = D.apply_operator(ctx, u)
    assert rel(got, G[name + "/Au"]) <= RTOL
    b = np.random.default_rng(4).uniform(-1.0, 1.0, ctx.ndofs)
    r = D.residual(ctx, u, b, np.empty(ctx.ndofs))
    assert rel(r, b - G[name + "/Au"]) <= RTOL


@pytest.mark.parametrize("name", CASES)
def test_distorted_operator_symmetric(name):
    ctx, _ = _ctx(name)
    g = torch.Generator(device="cuda").manual_seed(5)
    u = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    v = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    au, av = D.apply_operator(ctx, u), D.apply_operator(ctx, v)
    s1, s2 = float(v @ au), float(u @ av)
    assert abs(s1 - s2) <= 1e-12 * max(1.0, abs(s1))
    assert float(u @ au) > 0.0
