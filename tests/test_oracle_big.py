"""Pin the CPU oracle on the sizes beyond the templated kernels: vertex
patches of degree 8..15 and one-dimensional levels, against the reference's
own outputs (tests/golden/make_golden_big.py)."""
import pytest

from _common import golden_big, inputs, rel, RTOL
from oracle.sipg_oracle import OracleLevel

G = golden_big()
OPS = sorted({k.split("/")[0] for k in G if k.startswith("op_")})
STEPS = sorted({k.split("/")[0] for k in G if k.startswith("sm_")})


@pytest.mark.parametrize("name", OPS)
def test_oracle_operator_1d_matches_reference(name):
    _, d, k, nc = name.split("_")
    d, k, nc = int(d[0]), int(k[1:]), int(nc[1:])
    lvl = OracleLevel((nc,) * d, k)
    x0, b = inputs(lvl.ndofs)
    assert rel(lvl.apply(x0), G[name + "/Ax"]) <= RTOL
    assert rel(lvl.residual(x0, b), G[name + "/res"]) <= RTOL


@pytest.mark.parametrize("name", STEPS)
def test_oracle_step_matches_reference(name):
    kind = name.split("_")[1]
    d, nc, k, om, rev = G[name + "/meta"]
    lvl = OracleLevel((int(nc),) * int(d), int(k))
    x0, b = inputs(lvl.ndofs)
    x = lvl.smooth(kind, float(om), x0, b, reverse=bool(rev))
    assert rel(x, G[name + "/x"]) <= RTOL
    assert rel(x - x0, G[name + "/x"] - x0) <= 1e-11
