"""Distorted (multilinear) meshes at the degrees beyond the register
kernels: 2D k = 8..15 and 3D k = 5..15 run the shared-memory operator and
surrogate cell-solve kernels (csrc/dist_op.cu; 3D k = 15 with the face phase
aliased onto the volume buffers).  Against the reference's own outputs
(tests/golden/make_golden_dist_big.py): operator, residual, surrogate cell
solver set, one ACS and one MCS step.  Tolerance: rel L2 <= 1e-12."""
import os

import numpy as np
import pytest
import torch

from _common import rel, RTOL

from paper_1910_11239_b200 import distorted as D, mesh
from paper_1910_11239_b200.basis import Basis1D
from paper_1910_11239_b200.smoothers import SmootherConfig

pytestmark = pytest.mark.gpu
G = dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                              "golden_dist_big.npz")))
CASES = sorted({k.split("/")[0] for k in G if k.startswith("dbig_")})


def _ctx(name):
    d, coarse, level, k = (int(v) for v in G[name + "/meta"])
    h = D.distort(mesh.build_hierarchy(d, coarse, level), 0.25, 2024)
    return D.DistortedContext(h.levels[level], Basis1D.make(k), 4.0), h.levels[level]


@pytest.mark.parametrize("name", CASES)
def test_distorted_operator_matches_reference_big(name):
    ctx, lvl = _ctx(name)
    assert np.array_equal(lvl.vertex_grid, G[name + "/grid"])
    u = np.random.default_rng(3).uniform(-1.0, 1.0, ctx.ndofs)
    assert rel(D.apply_operator(ctx, u), G[name + "/Au"]) <= RTOL
    b = np.random.default_rng(4).uniform(-1.0, 1.0, ctx.ndofs)
    r = D.residual(ctx, u, b, np.empty(ctx.ndofs))
    assert rel(r, b - G[name + "/Au"]) <= RTOL


@pytest.mark.parametrize("name", CASES)
def test_distorted_operator_symmetric_big(name):
    ctx, _ = _ctx(name)
    g = torch.Generator(device="cuda").manual_seed(5)
    u = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    v = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    au, av = D.apply_operator(ctx, u), D.apply_operator(ctx, v)
    s1, s2 = float(v @ au), float(u @ av)
    assert abs(s1 - s2) <= 1e-12 * max(1.0, abs(s1))
    assert float(u @ au) > 0.0


@pytest.mark.parametrize("name", CASES)
def test_surrogate_cell_solves_and_steps_match_reference_big(name):
    ctx, _ = _ctx(name)
    n = ctx.ndofs
    r = np.random.default_rng(5).uniform(-1.0, 1.0, n)
    x = np.zeros(n)
    D.SurrogateCellSolverSet(ctx).solve_partitioned(x, r, None, 0.5)
    assert rel(x, G[name + "/cellset"]) <= RTOL
    b = np.random.default_rng(6).uniform(-1.0, 1.0, n)
    for kind, om in (("acs", 0.5), ("mcs", 0.75)):
        sm = D.DistortedSmoother(ctx, SmootherConfig(kind=kind, omega=om))
        x = np.random.default_rng(7).uniform(-1.0, 1.0, n)
        sm.smooth(x, b)
        assert rel(x, G[name + f"/{kind}"]) <= RTOL
