"""Pin the CPU oracle against golden vectors produced by the reference.

The oracle (oracle/sipg_oracle.py) is the checker for every GPU parity test,
so it must itself agree with the reference on the reference's own outputs
(tests/golden/make_golden.py) before it is trusted.
"""
import numpy as np
import pytest

from _common import golden, inputs, rel, RTOL
from oracle.sipg_oracle import OracleLevel, geneig

G = golden()

OPS = sorted({k.split("/")[0] for k in G if k.startswith("op_")})
STEPS = sorted({k.split("/")[0] for k in G if k.startswith("sm_")})


@pytest.mark.parametrize("name", OPS)
def test_oracle_operator_matches_reference(name):
    _, d, k, nc = name.split("_")
    d, k, nc = int(d[0]), int(k[1:]), int(nc[1:])
    lvl = OracleLevel((nc,) * d, k)
    x0, b = inputs(lvl.ndofs)
    assert rel(lvl.apply(x0), G[name + "/Ax"]) <= RTOL
    assert rel(lvl.residual(x0, b), G[name + "/res"]) <= RTOL


@pytest.mark.parametrize("name", STEPS)
def test_oracle_smoothing_step_matches_reference(name):
    kind = name.split("_")[1]
    d, nc, k, om, rev = G[name + "/meta"]
    lvl = OracleLevel((int(nc),) * int(d), int(k))
    x0, b = inputs(lvl.ndofs)
    x = lvl.smooth(kind, float(om), x0, b, reverse=bool(rev))
    assert rel(x, G[name + "/x"]) <= RTOL
    # the correction itself, not only the sum with x0
    assert rel(x - x0, G[name + "/x"] - x0) <= 1e-11


@pytest.mark.parametrize("name", ["map_3d_q3_n4", "map_2d_q2_n5", "map_3d_q1_n5"])
def test_oracle_patch_maps_bit_exact(name):
    _, d, k, nc = name.split("_")
    lvl = OracleLevel((int(nc[1:]),) * int(d[0]), int(k[1:]))
    gi = lvl.patch_map(lvl.patch_vertices())
    assert np.array_equal(gi, G[name + "/gidx"])


@pytest.mark.parametrize("name,d,nc", [("col_3d_n8", 3, 8), ("col_2d_n7", 2, 7),
                                       ("col_3d_n5", 3, 5)])
def test_oracle_colours_bit_exact(name, d, nc):
    lvl = OracleLevel((nc,) * d, 1)
    cols = lvl.colours("avs")
    assert np.array_equal(np.concatenate(cols), G[name + "/patch_order"])
    assert np.array_equal(np.concatenate([np.full(len(s), c) for c, s in enumerate(cols)]),
                          G[name + "/patch_colour"])
    rb = lvl.colours("mcs")
    assert np.array_equal(np.concatenate(rb), G[name + "/rb_order"])


def test_oracle_solver_sets_match_reference():
    lvl = OracleLevel((4, 4, 4), 3)
    _, r = inputs(lvl.ndofs, 7)
    x = np.zeros(lvl.ndofs)
    lvl.cell_solve(x, r, 1.0)
    assert rel(x, G["cellset_3d_q3_n4/x"]) <= RTOL
    x = np.zeros(lvl.ndofs)
    lvl.cell_solve(x, r, 0.5, np.array([0, 5, 21, 63]))
    assert rel(x, G["cellset_sub_3d_q3_n4/x"]) <= RTOL
    x = np.zeros(lvl.ndofs)
    lvl.patch_solve(x, r, 1.0, safe=True)
    assert rel(x, G["patchset_3d_q3_n4/x"]) <= RTOL


@pytest.mark.parametrize("k", [1, 2, 3, 5, 7, 15])
def test_oracle_1d_factors_match_reference(k):
    lvl = OracleLevel((8,), k)
    s = lvl.s
    for digit in range(4):
        pre = f"f1d_k{k}_d{digit}/"
        assert np.allclose(s.cell_stiffness(digit), G[pre + "cell_A"], rtol=1e-14, atol=1e-12)
        assert np.allclose(s.mass, G[pre + "cell_M"], rtol=1e-14, atol=1e-16)
        _, lam = geneig(s.cell_stiffness(digit), s.mass)
        assert rel(lam, G[pre + "cell_lam"]) <= 1e-13
        if k <= 7:
            a, m = s.patch_matrices(digit)
            assert np.allclose(a, G[pre + "patch_A"], rtol=1e-14, atol=1e-12)
            assert np.allclose(m, G[pre + "patch_M"], rtol=1e-14, atol=1e-16)


def test_oracle_dense_operator_is_spd():
    lvl = OracleLevel((3, 3), 2)
    a = lvl.dense()
    assert np.allclose(a, a.T, atol=1e-12 * np.abs(a).max())
    assert np.linalg.eigvalsh(a).min() > 0


def test_oracle_box_levels_are_consistent():
    """A box (3,3,5) is the cube algorithm with per-direction counts: the
    operator stays symmetric and the AVS step is linear in b."""
    lvl = OracleLevel((3, 3, 5), 1, h=1.0 / 3)
    x0, b = inputs(lvl.ndofs, 3)
    u, v = inputs(lvl.ndofs, 5)
    assert abs(u @ lvl.apply(v) - v @ lvl.apply(u)) <= 1e-12 * abs(u @ lvl.apply(u))
    s1 = lvl.smooth("avs", 0.25, x0, b)
    s2 = lvl.smooth("avs", 0.25, x0, 2 * b)
    s0 = lvl.smooth("avs", 0.25, x0, 0 * b)
    assert rel(s2 - s0, 2 * (s1 - s0)) <= 1e-13
