"""The drop-in claim of INTEGRATION.md section 1, tested against the
unmodified reference (`dgmg` from baseline/_ref or /root/reference):

- `make_context` takes the reference's own `MeshLevel` / `Basis1D` and
  builds the same device tables as from this package's objects (CPU);
- `SubdomainMap` / `restrict_to_subdomain` / `scatter_add_subdomain`
  (`smoothers.py:72-100`) give the reference's index
  lists and results (CPU for cells, GPU for the patch maps);
- a reference `dgmg.multigrid.VCycle` whose level smoothers are replaced by
  the device smoothers (`multigrid.py:334-343` calls only
  `.smooth(x, b, reverse)`) gives the reference's `VCycle.apply` to 1e-12
  (GPU).
"""
import numpy as np
import pytest

from _common import RTOL, inputs, ref_dgmg, rel

import paper_1910_11239_b200 as dg
from paper_1910_11239_b200 import smoothers as S

R = ref_dgmg()
needs_ref = pytest.mark.skipif(R is None, reason="reference dgmg not available")


def _ref_mods():
    from dgmg import dgop, fastdiag, mesh, multigrid, polybasis, smoothers
    return dgop, fastdiag, mesh, multigrid, polybasis, smoothers


@needs_ref
@pytest.mark.parametrize("d,nc,k", [(2, 4, 3), (3, 4, 2), (3, 2, 5)])
def test_make_context_accepts_reference_level_and_basis(d, nc, k):
    dgop, _, mesh, _, polybasis, _ = _ref_mods()
    rlvl = mesh.build_hierarchy(d, nc, 0).levels[0]
    rbasis = polybasis.Basis1D.make(k)
    got = dg.make_context(rlvl, rbasis, 1.0)
    want = dg.make_context(dg.build_hierarchy(d, nc, 0).levels[0], dg.Basis1D.make(k), 1.0)
    assert got.layout == want.layout and got.ndofs == rlvl.ncells * (k + 1) ** d
    for name in ("mass", "adiag", "bg", "cell_z", "cell_invsum"):
        a, b = getattr(got.tables, name), getattr(want.tables, name)
        assert np.array_equal(np.asarray(a), np.asarray(b)), name
    # the reference's own context for the same level has the same dof count
    assert dgop.make_context(rlvl, rbasis, 1.0).ndofs == got.ndofs


@needs_ref
@pytest.mark.parametrize("d,nc,k", [(2, 3, 2), (3, 2, 3)])
def test_subdomain_map_for_cells_matches_reference(d, nc, k):
    dgop, _, mesh, _, polybasis, smoothers = _ref_mods()
    rctx = dgop.make_context(mesh.build_hierarchy(d, nc, 0).levels[0], polybasis.Basis1D.make(k), 1.0)
    ctx = dg.make_context(dg.build_hierarchy(d, nc, 0).levels[0], dg.Basis1D.make(k), 1.0)
    got = S.SubdomainMap.for_cells(ctx)
    want = smoothers.SubdomainMap.for_cells(rctx)
    assert len(got) == len(want)
    for a, b in zip(got.indices, want.indices):
        assert np.array_equal(a, b)


@needs_ref
def test_restrict_and_scatter_match_reference_with_repeats():
    _, _, _, _, _, smoothers = _ref_mods()
    rng = np.random.default_rng(3)
    idx = [rng.integers(0, 50, 17), np.arange(10), np.array([4, 4, 4, 9])]
    mine, theirs = S.SubdomainMap(idx), smoothers.SubdomainMap(idx)
    x = rng.uniform(-1, 1, 50)
    for j in range(3):
        assert np.array_equal(S.restrict_to_subdomain(mine, x, j),
                              smoothers.restrict_to_subdomain(theirs, x, j))
        loc = rng.uniform(-1, 1, idx[j].size)
        a, b = x.copy(), x.copy()
        S.scatter_add_subdomain(mine, loc, j, a, scale=0.3)
        smoothers.scatter_add_subdomain(theirs, loc, j, b, scale=0.3)
        assert np.array_equal(a, b)


# ------------------------------------------------------------------ GPU --
@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("d,nc,k", [(2, 4, 2), (3, 3, 3)])
def test_subdomain_map_for_patches_matches_reference(d, nc, k):
    import torch
    dgop, fastdiag, mesh, _, polybasis, smoothers = _ref_mods()
    rlvl = mesh.build_hierarchy(d, nc, 0).levels[0]
    rset = fastdiag.PatchSolverSet(rlvl, polybasis.Basis1D.make(k), 1.0,
                                   patches=mesh.enumerate_vertex_patches(rlvl))
    want = smoothers.SubdomainMap.for_patches(rset)
    ctx = dg.make_context(dg.build_hierarchy(d, nc, 0).levels[0], dg.Basis1D.make(k), 1.0)
    sm = dg.make_level_smoother(ctx, dg.Basis1D.make(k), dg.SmootherConfig(kind="avs", omega=0.25))
    got = S.SubdomainMap.for_patches(sm.set)
    assert len(got) == len(want)
    for a, b in zip(got.indices, want.indices):
        assert np.array_equal(a, b)
    # R_j on device tensors, and the adjoint identity <R_j x, y> = <x, R_j^T y>
    x0, y0 = inputs(ctx.ndofs, 5)
    xt = torch.from_numpy(x0).cuda()
    for j in (0, len(got) // 2, len(got) - 1):
        rx = S.restrict_to_subdomain(got, xt, j)
        assert np.array_equal(rx.cpu().numpy(), smoothers.restrict_to_subdomain(want, x0, j))
        y = y0[:rx.numel()]
        acc = torch.zeros_like(xt)
        S.scatter_add_subdomain(got, torch.from_numpy(y).cuda(), j, acc)
        assert abs(float(rx.cpu().numpy() @ y) - float(acc.cpu().numpy() @ x0)) <= 1e-13 * ctx.ndofs


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("kind,omega,d,k,nc,levels", [
    ("avs", 0.125, 3, 2, 2, 2), ("mvs", 1.0, 3, 3, 2, 1), ("acs", 0.7, 2, 3, 2, 3),
    ("mcs", 1.0, 2, 4, 4, 2)])
def test_device_smoothers_in_reference_vcycle(kind, omega, d, k, nc, levels):
    """A reference V-cycle with its level smoothers replaced by the device
    smoothers built from the reference's own contexts and basis
    (INTEGRATION.md section 1): the reference's residual, transfers and
    coarse solve stay; the preconditioner action equals the unpatched one."""
    dgop, _, mesh, multigrid, polybasis, smoothers = _ref_mods()
    basis = polybasis.Basis1D.make(k)
    ctxs = [dgop.make_context(lv, basis, 1.0) for lv in mesh.build_hierarchy(d, nc, levels).levels]
    mcfg = multigrid.MultigridConfig(smoother=smoothers.SmootherConfig(kind=kind, omega=omega))
    vc = multigrid.VCycle(ctxs, basis, mcfg)
    b = np.random.default_rng(11).uniform(-1, 1, ctxs[-1].ndofs)
    want = vc.apply(b)
    for ell in range(1, len(ctxs)):
        ctx = dg.make_context(ctxs[ell].level, basis, ctxs[ell].gamma_hat)
        vc.smoothers[ell] = dg.make_level_smoother(ctx, basis, dg.SmootherConfig(kind=kind, omega=omega))
    got = vc.apply(b)
    assert rel(got, want) <= RTOL
