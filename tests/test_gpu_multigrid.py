"""GPU parity of the multigrid / Krylov layer around the smoother (SURVEY
8(f) rows 1-2): the sm_100a transfer kernels, the device V-cycle and the
device CG, against the reference's golden vectors, the pinned oracle, and
the reference's own multigrid properties (`test_multigrid.py`)."""
import numpy as np
import pytest
import torch

from _common import golden_mg, rel, useed, RTOL

import paper_1910_11239_b200 as dg
from paper_1910_11239_b200 import dgop, krylov
from paper_1910_11239_b200 import multigrid as mg
from oracle.sipg_oracle import OracleVCycle, pcg as opcg, prolongate, restrict

pytestmark = pytest.mark.gpu
G = golden_mg()
TRS = sorted({k.split("/")[0] for k in G if k.startswith("tr_")})
VCS = sorted({k.split("/")[0] for k in G if k.startswith("vc_")})
CGS = sorted({k.split("/")[0] for k in G if k.startswith("cg_")})


def stack(d, coarse, levels, k, **kw):
    h = dg.build_hierarchy(d, coarse, levels)
    basis = dg.Basis1D.make(k)
    ctxs = [dg.make_context(lvl, basis, 1.0) for lvl in h.levels]
    return basis, ctxs, mg.VCycle(ctxs, basis, mg.MultigridConfig(**kw))


def transfer(d, nc, k):
    basis = dg.Basis1D.make(k)
    h = dg.build_hierarchy(d, nc, 1)
    ctxs = [dg.make_context(lvl, basis, 1.0) for lvl in h.levels]
    return ctxs, mg.LevelTransfer(mg.build_transfer(basis), ctxs[0], ctxs[1])


# ---------------------------------------------------------------- transfers --
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5, 6, 7, 15])
def test_build_transfer_matches_reference(k):
    pair = mg.build_transfer(dg.Basis1D.make(k))
    assert np.abs(pair.e0 - G[f"E_k{k}/e0"]).max() <= 1e-13
    assert np.abs(pair.e1 - G[f"E_k{k}/e1"]).max() <= 1e-13


@pytest.mark.parametrize("name", TRS)
def test_transfers_match_reference(name):
    _, d, k, nc = name.split("_")
    d, k, nc = int(d[0]), int(k[1:]), int(nc[1:])
    ctxs, tr = transfer(d, nc, k)
    xc = useed(ctxs[0].ndofs, 0)
    xf = useed(ctxs[1].ndofs, 1)
    p = np.empty(ctxs[1].ndofs)
    assert tr.prolongate(xc, p) is p
    assert rel(p, G[name + "/P"]) <= RTOL
    r = np.empty(ctxs[0].ndofs)
    assert tr.restrict(xf, r) is r
    assert rel(r, G[name + "/R"]) <= RTOL


@pytest.mark.parametrize("d,nc,k", [(3, 16, 5), (3, 8, 7), (2, 32, 3), (3, 4, 15),
                                    (3, 10, 2), (2, 7, 11), (3, 3, 9), (1, 33, 4)])
def test_transfers_match_oracle_at_size(d, nc, k):
    ctxs, tr = transfer(d, nc, k)
    xc = useed(ctxs[0].ndofs, 3)
    xf = useed(ctxs[1].ndofs, 4)
    dims = (nc,) * d
    xct = torch.from_numpy(xc).cuda()
    pt = torch.empty(ctxs[1].ndofs, dtype=torch.float64, device="cuda")
    tr.prolongate(xct, pt)
    assert rel(pt.cpu().numpy(), prolongate(dims, k, xc)) <= RTOL
    rt = torch.empty(ctxs[0].ndofs, dtype=torch.float64, device="cuda")
    tr.restrict(torch.from_numpy(xf).cuda(), rt)
    assert rel(rt.cpu().numpy(), restrict(dims, k, xf)) <= RTOL
    # fused accumulate = prolongate then add, bit for bit
    base = torch.from_numpy(xf).cuda()
    acc = base.clone()
    tr.prolongate(xct, acc, accumulate=True)
    assert torch.equal(acc, base + pt)


def test_transfer_properties():
    """`test_multigrid.py:68-120`: constants, adjointness, zero, SPD Gram."""
    ctxs, tr = transfer(2, 2, 3)
    out = np.empty(ctxs[1].ndofs)
    tr.prolongate(np.ones(ctxs[0].ndofs), out)
    assert np.allclose(out, 1.0, atol=1e-14)
    rng = np.random.default_rng(6)
    u = rng.standard_normal(ctxs[0].ndofs)
    v = rng.standard_normal(ctxs[1].ndofs)
    up = tr.prolongate(u, np.empty(ctxs[1].ndofs))
    vr = tr.restrict(v, np.empty(ctxs[0].ndofs))
    assert abs(up @ v - u @ vr) <= 1e-13 * max(1.0, abs(up @ v))
    ctxs, tr = transfer(2, 2, 1)
    z = np.empty(ctxs[0].ndofs)
    tr.restrict(np.zeros(ctxs[1].ndofs), z)
    assert np.all(z == 0.0)
    n0 = ctxs[0].ndofs
    gram = np.empty((n0, n0))
    for j in range(n0):
        e = np.zeros(n0)
        e[j] = 1.0
        gram[:, j] = tr.restrict(tr.prolongate(e, np.empty(ctxs[1].ndofs)), np.empty(n0))
    assert np.linalg.eigvalsh(0.5 * (gram + gram.T))[0] > 0.0


@pytest.mark.parametrize("dim,k", [(1, 3), (2, 2), (2, 4), (3, 2)])
def test_prolongation_polynomial_exactness(dim, k):
    """`test_multigrid.py:32-65`: polynomials of degree <= k are reproduced."""
    ctxs, tr = transfer(dim, 2, k)
    rng = np.random.default_rng(4)
    coef = rng.standard_normal((k + 1,) * dim)
    nodes = dg.Basis1D.make(k).nodes

    def interp(nc):
        n = k + 1
        idx = np.indices((nc,) * dim + (n,) * dim).reshape(2 * dim, -1)
        x = np.empty((idx.shape[1], dim))
        for t in range(dim):                 # canonical grid axes (c_d..c_1, i_d..i_1)
            x[:, t] = (idx[dim - 1 - t] + nodes[idx[2 * dim - 1 - t]]) / nc
        val = np.zeros(len(x))
        for ids in np.ndindex(*coef.shape):
            term = coef[ids]
            for t in range(dim):
                term = term * x[:, t] ** ids[t]
            val += term
        return val

    fine = np.empty(ctxs[1].ndofs)
    tr.prolongate(interp(2), fine)
    expect = interp(4)
    assert np.allclose(fine, expect, atol=1e-13 * max(1.0, np.abs(expect).max()))


# ---------------------------------------------------------------- coarse ----
@pytest.mark.parametrize("name,d,nc,k", [("cs_2d_q2_n4", 2, 4, 2), ("cs_3d_q3_n2", 3, 2, 3)])
def test_coarse_solvers_match_reference(name, d, nc, k):
    basis = dg.Basis1D.make(k)
    ctx = dg.make_context(dg.build_hierarchy(d, nc, 0).levels[0], basis, 1.0)
    b = useed(ctx.ndofs, 0)
    x = np.empty_like(b)
    cs = mg.CoarseSolver(ctx, basis, mg.MultigridConfig(coarse="direct"))
    assert cs.solve(b, x) is x and cs.mode == "direct"
    assert rel(x, G[name + "/direct"]) <= 1e-12
    x = np.empty_like(b)
    mg.CoarseSolver(ctx, basis, mg.MultigridConfig(coarse="chebyshev_cg")).solve(b, x)
    assert rel(x, G[name + "/cheb"]) <= 1e-7
    assert rel(x, G[name + "/direct"]) <= 1e-7


@pytest.mark.parametrize("d,dims,k", [(3, (2, 2, 2), 5), (3, (3, 2, 4), 3), (2, (8, 8), 4),
                                      (2, (5, 3), 7), (3, (1, 1, 1), 6), (1, (7,), 4),
                                      (3, (2, 2, 2), 15), (2, (32, 32), 3)])
def test_kronecker_fdm_coarse_solve_is_exact(d, dims, k):
    """Direct coarse solve on Cartesian levels (global fast diagonalisation,
    csrc/coarse.cu): A x = b to rounding, and equal to a dense solve with the
    assembled matrix (the reference's Cholesky / LU, `multigrid.py:169-195`)."""
    from paper_1910_11239_b200.mesh import MeshLevel
    lvl = MeshLevel(d, tuple(dims), 1.0 / dims[0])
    basis = dg.Basis1D.make(k)
    ctx = dg.make_context(lvl, basis, 1.0)
    cs = mg.CoarseSolver(ctx, basis, mg.MultigridConfig(coarse="direct"))
    assert cs.mode == "direct" and cs.direct_kind == "kronecker_fdm"
    b = torch.from_numpy(useed(ctx.ndofs, 3)).cuda()
    x = torch.empty_like(b)
    cs.solve(b, x)
    ax = dg.apply_operator(ctx, x)
    assert float((ax - b).norm() / b.norm()) <= 1e-11
    if ctx.ndofs <= 6000:
        a = dgop.assemble_dense(ctx, device="cuda")
        want = torch.linalg.solve(a, b)
        assert float((x - want).norm() / want.norm()) <= 1e-10


def test_mode_contract_matches_tensordot():
    g = torch.Generator("cuda").manual_seed(5)
    t = torch.rand((3, 5, 7, 4), dtype=torch.float64, device="cuda", generator=g)
    for ax, i in ((1, 6), (2, 2), (3, 9), (0, 4)):
        m = torch.rand((i, t.shape[ax]), dtype=torch.float64, device="cuda", generator=g)
        want = torch.movedim(torch.tensordot(t, m, dims=([ax], [1])), -1, ax)
        got = dgop.mode_contract(t, m, ax)
        assert got.shape == want.shape
        assert float((got - want).abs().max()) <= 1e-13
    with pytest.raises(ValueError):
        dgop.mode_contract(t, torch.zeros((2, 3), dtype=torch.float64, device="cuda"), 1)


def test_coarse_zero_rhs_and_dense_assembly():
    basis = dg.Basis1D.make(2)
    ctx = dg.make_context(dg.build_hierarchy(2, 2, 0).levels[0], basis, 1.0)
    x = np.empty(ctx.ndofs)
    mg.CoarseSolver(ctx, basis, mg.MultigridConfig()).solve(np.zeros(ctx.ndofs), x)
    assert np.allclose(x, 0.0, atol=1e-14)
    a_k = dgop.assemble_dense(ctx)
    a_m = dgop.assemble_dense(ctx, via="matvec")
    assert np.abs(a_k - a_m).max() <= 1e-12 * np.abs(a_k).max()


# ---------------------------------------------------------------- V-cycle ---
@pytest.mark.parametrize("name", VCS)
def test_vcycle_matches_reference(name):
    kind = name.split("_")[1]
    d, nc, lv, k, om, m, sym = G[name + "/meta"]
    cfg = dg.SmootherConfig(kind=kind, omega=float(om), m_pre=int(m), m_post=int(m),
                            symmetrize=bool(sym))
    _, ctxs, cyc = stack(int(d), int(nc), int(lv), int(k), smoother=cfg)
    b = useed(ctxs[-1].ndofs, 0)
    out = np.empty_like(b)
    assert cyc.apply(b, out) is out
    assert rel(out, G[name + "/x"]) <= 1e-11
    # device tensors in and out give the same result
    xt = cyc.apply(torch.from_numpy(b).cuda())
    assert rel(xt.cpu().numpy(), out) <= 1e-14


@pytest.mark.parametrize("kind,omega,m", [("avs", 0.25, 1), ("mvs", 1.0, 1), ("acs", 0.7, 1)])
def test_vcycle_matches_oracle_3d(kind, omega, m):
    cfg = dg.SmootherConfig(kind=kind, omega=omega, m_pre=m, m_post=m)
    _, ctxs, cyc = stack(3, 2, 2, 3, smoother=cfg)
    b = useed(ctxs[-1].ndofs, 5)
    ocyc = OracleVCycle(3, 2, 2, 3, kind, omega, m, m)
    assert rel(cyc.apply(b), ocyc.apply(b)) <= 1e-11


def test_vcycle_linearity_and_symmetry():
    """`test_multigrid.py:133-172`."""
    cfg = dg.SmootherConfig(kind="acs", omega=0.7)
    _, ctxs, cyc = stack(2, 2, 1, 2, smoother=cfg)
    n = ctxs[1].ndofs
    rng = np.random.default_rng(8)
    b1, b2 = rng.standard_normal(n), rng.standard_normal(n)
    x1 = cyc.apply(b1).copy()
    x2 = cyc.apply(b2).copy()
    x12 = cyc.apply(0.7 * b1 - 1.3 * b2)
    assert np.allclose(x12, 0.7 * x1 - 1.3 * x2, atol=1e-11 * max(1.0, np.abs(x12).max()))
    for kind, om, sym in (("acs", 0.7, False), ("mvs", 1.0, True)):
        _, ctxs, cyc = stack(2, 2, 1, 2, smoother=dg.SmootherConfig(kind=kind, omega=om,
                                                                  symmetrize=sym))
        s1 = cyc.apply(b1) @ b2
        s2 = b1 @ cyc.apply(b2)
        assert abs(s1 - s2) <= 1e-10 * max(1.0, abs(s1))


def test_vcycle_level0_is_coarse_solve():
    _, ctxs, cyc = stack(2, 2, 1, 2)
    rng = np.random.default_rng(7)
    b = rng.standard_normal(ctxs[0].ndofs)
    x = np.zeros(ctxs[0].ndofs)
    cyc.vcycle(0, x, b)
    a = dgop.assemble_dense(ctxs[0])
    assert np.linalg.norm(a @ x - b) <= 1e-10 * np.linalg.norm(b)


@pytest.mark.parametrize("kind,omega,m", [("acs", 0.7, 1), ("mcs", 1.0, 1), ("avs", 0.25, 2),
                                          ("mvs", 1.0, 1)])
def test_vcycle_fixed_point_converges(kind, omega, m):
    """`test_multigrid.py:175-203`."""
    cfg = dg.SmootherConfig(kind=kind, omega=omega, m_pre=m, m_post=m)
    _, ctxs, cyc = stack(2, 2, 3, 3, smoother=cfg)
    ctx = ctxs[-1]
    rng = np.random.default_rng(11)
    b = rng.standard_normal(ctx.ndofs)
    x = np.zeros(ctx.ndofs)
    norms = [np.linalg.norm(b)]
    for _ in range(5):
        x += cyc.apply(b - dg.apply_operator(ctx, x))
        norms.append(np.linalg.norm(b - dg.apply_operator(ctx, x)))
    assert all(norms[i + 1] < norms[i] for i in range(5))
    assert norms[5] < 0.25 * norms[0]


# ---------------------------------------------------------------- Krylov ----
@pytest.mark.parametrize("name", CGS)
def test_pcg_vcycle_matches_reference(name):
    """Residual history and fractional iteration count of V-cycle CG (the
    quantity of acceptance criteria 3-5) equal the reference's."""
    kind = name.split("_")[1]
    d, nc, lv, k, om = G[name + "/meta"]
    _, ctxs, cyc = stack(int(d), int(nc), int(lv), int(k),
                         smoother=dg.SmootherConfig(kind=kind, omega=float(om)))
    ctx = ctxs[-1]
    b = useed(ctx.ndofs, 0)
    res = krylov.pcg(lambda x, o: dg.apply_operator(ctx, x, out=o), b,
                     lambda r, o: cyc.apply(r, o), delta_red=1e-8, max_it=100)
    ref = G[name + "/history"]
    assert res.converged and len(res.history) == len(ref)
    assert np.allclose(res.history, ref, rtol=1e-7, atol=0)
    nu, it = G[name + "/nu_frac"]
    assert res.iterations == int(it) and abs(res.nu_frac - nu) <= 1e-6
    assert isinstance(res.x, np.ndarray) and rel(res.x, G[name + "/x"]) <= 1e-9


def test_pcg_and_gmres_on_device_tensors():
    cfg = dg.SmootherConfig(kind="mvs", omega=1.0)
    _, ctxs, cyc = stack(3, 2, 2, 2, smoother=cfg)
    ctx = ctxs[-1]
    b = torch.from_numpy(useed(ctx.ndofs, 2)).cuda()
    op = lambda x, o: dg.apply_operator(ctx, x, out=o)  # noqa: E731
    pc = lambda r, o: cyc.apply(r, o)  # noqa: E731
    res = krylov.pcg(op, b, pc, delta_red=1e-10, max_it=50)
    assert res.converged and isinstance(res.x, torch.Tensor)
    r = b - dg.apply_operator(ctx, res.x)
    assert float(torch.linalg.vector_norm(r)) <= 1e-10 * float(torch.linalg.vector_norm(b)) * 1.01
    gm = krylov.pgmres(op, b, pc, delta_red=1e-10, max_it=50)
    assert gm.converged
    assert rel(gm.x.cpu().numpy(), res.x.cpu().numpy()) <= 1e-8
    # oracle CG with the oracle V-cycle: same iteration count
    ocyc = OracleVCycle(3, 2, 2, 2, "mvs", 1.0)
    top = ocyc.levels[-1]
    _, hist = opcg(top.apply, b.cpu().numpy(), ocyc.apply, 1e-10, 50)
    assert len(hist) == len(res.history)


def test_fused_cg_kernels_match_torch():
    from paper_1910_11239_b200.krylov import _Fused
    for n in (1, 7, 1000, 1 << 20, 3 * (1 << 20) + 1):
        g = torch.Generator(device="cuda").manual_seed(n)
        x, r, p, ap = (torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
                       for _ in range(4))
        f = _Fused(n)
        x0, r0 = x.clone(), r.clone()
        rr = f.update(x, r, p, ap, 0.37)
        assert torch.allclose(x, x0 + 0.37 * p, rtol=1e-15, atol=1e-15)
        assert torch.allclose(r, r0 - 0.37 * ap, rtol=1e-15, atol=1e-15)
        assert abs(rr - float(r @ r)) <= 1e-12 * max(1.0, abs(rr))
        assert abs(f.dot(p, ap) - float(p @ ap)) <= 1e-12 * max(1.0, float(p @ ap))
        z = ap.clone()
        p0 = p.clone()
        f.direction(p, z, -0.5)
        assert torch.allclose(p, z - 0.5 * p0, rtol=1e-15, atol=1e-15)
        # deterministic reductions
        assert f.dot(p, ap) == f.dot(p, ap)


@pytest.mark.parametrize("name", sorted({k.split("/")[0] for k in G if k.startswith("rhs_")}))
def test_compute_rhs_matches_reference(name):
    """`dgop.compute_rhs` (`dgop.py:800-871`): volume source and Nitsche
    boundary data contracted on the device, against the reference's vector."""
    from _common import rhs_f, rhs_g
    _, d, k, nc = name.split("_")
    d, k, nc = int(d[0]), int(k[1:]), int(nc[1:])
    basis = dg.Basis1D.make(k)
    ctx = dg.make_context(dg.build_hierarchy(d, nc, 0).levels[0], basis, 1.0)
    got = dgop.compute_rhs(ctx, rhs_f, rhs_g)
    assert got.shape == (ctx.ndofs,)
    assert rel(got, G[name + "/rhs"]) <= 1e-13


@pytest.mark.parametrize("d,nc,lv,k,kind,om", [(3, 2, 2, 3, "avs", 0.125), (2, 4, 2, 4, "acs", 0.7),
                                               (3, 2, 2, 2, "mvs", 1.0), (1, 3, 3, 3, "avs", 0.5)])
def test_vcycle_zero_guess_shortcut_is_exact(d, nc, lv, k, kind, om, monkeypatch):
    """The first pre-smoothing step of a V-cycle level starts from x = 0, where
    r = b - A 0 = b bit for bit: the additive kinds skip that residual launch
    (`LevelSmoother.smooth_from_zero`).  Same cycle as without the shortcut:
    bitwise for ACS (and MVS, which takes the ordinary step), to rounding for
    AVS, whose one-launch path sums a DoF's updates in arbitrary order."""
    cfg = dg.SmootherConfig(kind=kind, omega=om, m_pre=2, m_post=1)
    out = {}
    for v in ("0", "1"):
        monkeypatch.setenv("DGB_ZERO_GUESS", v)
        _, ctxs, cyc = stack(d, nc, lv, k, smoother=cfg)
        b = torch.from_numpy(useed(ctxs[-1].ndofs, 0)).cuda()
        out[v] = cyc.apply(b, torch.empty_like(b)).cpu().numpy()
    if kind == "avs":
        assert rel(out["1"], out["0"]) <= 1e-14
    else:
        assert np.array_equal(out["0"], out["1"])
    # and a single step: smooth_from_zero == smooth on a zero vector
    ctx = ctxs[-1]
    sm = cyc.smoothers[len(ctxs) - 1]
    x1 = torch.zeros(ctx.ndofs, dtype=torch.float64, device="cuda")
    x2 = torch.zeros_like(x1)
    monkeypatch.setenv("DGB_ZERO_GUESS", "1")
    sm.smooth_from_zero(x1, b)
    sm.smooth(x2, b)
    if kind == "avs":
        assert float((x1 - x2).norm() / x2.norm()) <= 1e-14
    else:
        assert torch.equal(x1, x2)
    # with the deterministic AVS order requested the shortcut steps aside
    if kind == "avs":
        monkeypatch.setenv("DGB_AVS_ATOMIC", "0")
        x3 = torch.zeros_like(x1)
        x4 = torch.zeros_like(x1)
        sm.smooth_from_zero(x3, b)
        sm.smooth(x4, b)
        assert torch.equal(x3, x4)
