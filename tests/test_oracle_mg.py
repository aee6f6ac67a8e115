"""Pin the multigrid / Krylov part of the CPU oracle
against golden vectors produced by the reference itself
(tests/golden/make_golden_mg.py), plus the reference's own transfer
properties (`test_multigrid.py:21-120`)."""
import numpy as np
import pytest

from _common import golden_mg, rel, useed
from oracle.sipg_oracle import (OracleLevel, OracleVCycle, embeddings, pcg, prolongate,
                                restrict)

G = golden_mg()
TRS = sorted({k.split("/")[0] for k in G if k.startswith("tr_")})
VCS = sorted({k.split("/")[0] for k in G if k.startswith("vc_")})
CGS = sorted({k.split("/")[0] for k in G if k.startswith("cg_")})


def _tr(name):
    _, d, k, nc = name.split("_")
    return int(d[0]), int(k[1:]), int(nc[1:])


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7, 15])
def test_oracle_embeddings_match_reference(k):
    e0, e1 = embeddings(k)
    assert np.abs(e0 - G[f"E_k{k}/e0"]).max() <= 1e-13
    assert np.abs(e1 - G[f"E_k{k}/e1"]).max() <= 1e-13


@pytest.mark.parametrize("name", TRS)
def test_oracle_transfers_match_reference(name):
    d, k, nc = _tr(name)
    n = k + 1
    dims = (nc,) * d
    xc = useed(nc ** d * n ** d, 0)
    xf = useed((2 * nc) ** d * n ** d, 1)
    assert rel(prolongate(dims, k, xc), G[name + "/P"]) <= 1e-13
    assert rel(restrict(dims, k, xf), G[name + "/R"]) <= 1e-13


def test_oracle_transfer_adjoint_and_constants():
    dims, k = (2, 3), 3
    rng = np.random.default_rng(6)
    u = rng.standard_normal(6 * 16)
    v = rng.standard_normal(24 * 16)
    assert abs(prolongate(dims, k, u) @ v - u @ restrict(dims, k, v)) <= 1e-12
    assert np.allclose(prolongate(dims, k, np.ones(6 * 16)), 1.0, atol=1e-14)


@pytest.mark.parametrize("name", VCS)
def test_oracle_vcycle_matches_reference(name):
    kind = name.split("_")[1]
    d, nc, lv, k, om, m, sym = G[name + "/meta"]
    cyc = OracleVCycle(int(d), int(nc), int(lv), int(k), kind, float(om), int(m), int(m),
                       bool(sym))
    b = useed(cyc.levels[-1].ndofs, 0)
    assert rel(cyc.apply(b), G[name + "/x"]) <= 1e-11


@pytest.mark.parametrize("name", CGS)
def test_oracle_pcg_history_matches_reference(name):
    kind = name.split("_")[1]
    d, nc, lv, k, om = G[name + "/meta"]
    cyc = OracleVCycle(int(d), int(nc), int(lv), int(k), kind, float(om))
    top = cyc.levels[-1]
    b = useed(top.ndofs, 0)
    x, hist = pcg(top.apply, b, cyc.apply, 1e-8, 100)
    ref = G[name + "/history"]
    assert len(hist) == len(ref)
    assert np.allclose(hist, ref, rtol=1e-7, atol=0)
    assert rel(x, G[name + "/x"]) <= 1e-9


def test_oracle_dense_coarse_solve_matches_reference():
    lvl = OracleLevel((4, 4), 2)
    b = useed(lvl.ndofs, 0)
    assert rel(np.linalg.solve(lvl.dense(), b), G["cs_2d_q2_n4/direct"]) <= 1e-12
    lvl = OracleLevel((2, 2, 2), 3)
    b = useed(lvl.ndofs, 0)
    assert rel(np.linalg.solve(lvl.dense(), b), G["cs_3d_q3_n2/direct"]) <= 1e-12
