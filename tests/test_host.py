"""CPU tests of the host side: 1D setup, tables, index maps, colourings,
config validation, work model, and that the C-ABI library loads and exports
every symbol the header declares (no compute without a GPU)."""
import ctypes
import os
import re
import sys

import numpy as np
import pytest

from _common import golden, have_reference, rel, REF_SRC

import paper_1910_11239_b200 as dg
from paper_1910_11239_b200 import basis as B
from paper_1910_11239_b200 import mesh as M
from paper_1910_11239_b200 import tables as T
from paper_1910_11239_b200 import flops as F

G = golden()
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------ C ABI --
def _header_symbols():
    src = open(os.path.join(ROOT, "include", "dgmg_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\*\s]+?\b(dg_\w+)\s*\(", src, re.M)))


def test_header_declares_the_abi():
    syms = _header_symbols()
    for s in ("dg_level_create", "dg_residual", "dg_apply", "dg_cell_fdm", "dg_patch_fdm",
              "dg_smooth", "dg_patch_gather_map", "dg_last_error"):
        assert s in syms


def test_library_loads_and_exports_every_symbol():
    from paper_1910_11239_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        import __graft_entry__
        __graft_entry__.build()
    lib = _lib.load()
    for s in _header_symbols():
        assert hasattr(lib, s), s
    assert set(_header_symbols()) == set(_lib.EXPORTS)
    assert lib.dg_version() == 1


def test_library_rejects_bad_arguments_without_gpu():
    from paper_1910_11239_b200 import _lib
    lib = _lib.load()
    h = ctypes.c_void_p()
    desc = _lib.LevelDesc()
    desc.dim = 4
    rc = lib.dg_level_create(ctypes.byref(desc), ctypes.byref(_lib.Tables()), ctypes.byref(h))
    assert rc == _lib.DG_EUNSUPPORTED
    assert b"dim" in lib.dg_last_error()
    assert lib.dg_level_create(None, None, None) == _lib.DG_EINVAL
    with pytest.raises(NotImplementedError):
        _lib.check(_lib.DG_EUNSUPPORTED)
    with pytest.raises(ValueError):
        _lib.check(_lib.DG_EINVAL)
    with pytest.raises(dg.SingularLocalSolverError):
        _lib.check(_lib.DG_ESINGULAR)


@pytest.mark.parametrize("d,nc", [(3, (1025, 4, 4)), (3, (4, 4, 2048)), (2, (32769, 2, 1))])
def test_level_create_rejects_levels_the_packed_lists_cannot_hold(d, nc):
    """Colour lists pack global coordinates in 10 (3D) / 15 (2D) bits: larger
    levels are refused before any allocation."""
    from paper_1910_11239_b200 import _lib
    lib = _lib.load()
    desc = _lib.LevelDesc()
    desc.dim, desc.degree = d, 1
    for t in range(3):
        desc.ncells[t] = nc[t]
    desc.z_begin, desc.z_count = 0, nc[d - 1]
    h = ctypes.c_void_p()
    rc = lib.dg_level_create(ctypes.byref(desc), ctypes.byref(_lib.Tables()), ctypes.byref(h))
    assert rc == _lib.DG_EUNSUPPORTED
    assert b"cells per direction" in lib.dg_last_error()


@pytest.mark.parametrize("starts,nz,want", [
    ([0, 4, 8, 9], 11, [0, 4, 8, 11]),          # ..., 1-layer chunk, 2-layer tail
    ([0, 8, 16, 17, 19], 21, [0, 8, 16, 19, 21]),
    ([0, 4, 8, 12], 13, [0, 4, 8, 13]),         # 1-layer last chunk
    ([0, 2, 4], 6, [0, 2, 4, 6]),
    ([0], 3, [0, 3]),
])
def test_pipeline_chunks_are_at_least_two_layers(starts, nz, want):
    from paper_1910_11239_b200.smoothers import _min2_chunks
    got = _min2_chunks(starts, nz)
    assert got == want
    assert all(b - a >= 2 for a, b in zip(got, got[1:]))


# --------------------------------------------------------------- 1D setup --
@pytest.mark.parametrize("k", [1, 2, 3, 5, 7, 15])
def test_host_1d_factors_match_reference(k):
    basis = B.Basis1D.make(k)
    h = 1.0 / 8
    for digit in range(4):
        pre = f"f1d_k{k}_d{digit}/"
        m, a = B.cell_factors(basis, h, bool(digit & 1), bool(digit & 2))
        assert np.array_equal(a, G[pre + "cell_A"]) or np.allclose(a, G[pre + "cell_A"],
                                                                   rtol=1e-15, atol=1e-13)
        assert np.allclose(m, G[pre + "cell_M"], rtol=1e-15, atol=1e-17)
        z, lam = B.sym_eig(a, m)
        assert rel(lam, G[pre + "cell_lam"]) <= 1e-14
        assert np.allclose(z.T @ a @ z, np.diag(lam), atol=1e-9 * lam.max())
        assert np.allclose(z.T @ m @ z, np.eye(k + 1), atol=1e-11)
        if k <= 7:
            pm, pa = B.patch_factors(basis, h, h, bool(digit & 1), bool(digit & 2))
            assert np.allclose(pa, G[pre + "patch_A"], rtol=1e-15, atol=1e-13)
            assert np.allclose(pm, G[pre + "patch_M"], rtol=1e-15, atol=1e-17)
            _, plam = B.sym_eig(pa, pm)
            assert rel(plam, G[pre + "patch_lam"]) <= 1e-14


def test_basis_nodes_and_boundary_tables():
    b = B.Basis1D.make(5)
    assert np.array_equal(b.nodes, G["basis_k5/nodes"])
    assert np.allclose(b.bg, G["basis_k5/bg"], rtol=1e-15, atol=1e-12)
    # nodal endpoints exactly: the device coupling relies on bv0 = e_0, bv1 = e_n-1
    assert np.array_equal(b.bv[0], np.eye(6)[0])
    assert np.array_equal(b.bv[1], np.eye(6)[5])
    with pytest.raises(ValueError):
        B.gl_nodes(0)
    assert dg.dgop.penalty(1.0, 3, 1.0, 1.0) == pytest.approx(24.0)
    assert dg.dgop.penalty(4.0, 3, 1.0, 1.0) == pytest.approx(96.0)


def test_tables_classes_and_inverse_sums():
    basis = B.Basis1D.make(2)
    tab = T.build_tables(basis, 0.25, (4, 4, 4))
    n, m = 3, 6
    # interior cell class code 0 and boundary classes present; absent ones zero
    for code in range(64):
        digs = [(code >> (2 * t)) & 3 for t in range(3)]
        present = all(dd != 3 for dd in digs)
        assert (np.abs(tab.cell_invsum[code]).sum() > 0) == present
        if present:
            lam = [tab.cell_lam[dd] for dd in digs]
            want = 1.0 / (lam[0][None, None, :] + lam[1][None, :, None] + lam[2][:, None, None])
            assert np.allclose(tab.cell_invsum[code].reshape(n, n, n), want, rtol=1e-15)
    assert tab.patch_invsum.shape == (64, m ** 3)
    assert T.patch_digits(2) == [3] and T.patch_digits(3) == [1, 2] and T.patch_digits(5) == [0, 1, 2]
    assert T.cell_digits(1) == [3] and T.cell_digits(2) == [1, 2]
    with pytest.raises(T.SingularLocalSolverError):
        T.inverse_sum([np.array([-1.0, 0.5]), np.array([0.2, 0.3])])


# ------------------------------------------------------------ index maps --
@pytest.mark.parametrize("name,d,nc", [("col_3d_n8", 3, 8), ("col_2d_n7", 2, 7),
                                       ("col_3d_n5", 3, 5)])
def test_structured_colours_bit_exact(name, d, nc):
    lvl = M.build_hierarchy(d, nc, 0).levels[0]
    cp = M.color_patches_structured(lvl)
    assert np.array_equal(np.concatenate(cp.sets), G[name + "/patch_order"])
    assert np.array_equal(np.concatenate([np.full(len(s), c) for c, s in enumerate(cp.sets)]),
                          G[name + "/patch_colour"])
    assert cp.validate_cover()
    rb = M.color_cells_redblack(lvl)
    assert np.array_equal(np.concatenate(rb.sets), G[name + "/rb_order"])
    assert [len(s) for s in rb.sets] == list(G[name + "/rb_sizes"])


@pytest.mark.parametrize("name", ["map_3d_q3_n4", "map_2d_q2_n5", "map_3d_q1_n5"])
def test_patch_cells_bit_exact(name):
    _, d, k, nc = name.split("_")
    lvl = M.build_hierarchy(int(d[0]), int(nc[1:]), 0).levels[0]
    assert np.array_equal(M.enumerate_vertex_patches(lvl).cells, G[name + "/cells"])


def test_mesh_counts_and_boxes():
    lvl = M.build_hierarchy(3, 2, 3).levels[3]
    assert lvl.ncells == 4096 and len(M.enumerate_vertex_patches(lvl)) == 3375
    assert len(M.color_patches_structured(lvl).sets) == 16
    assert len(M.color_patches_structured(M.build_hierarchy(2, 8, 0).levels[0]).sets) == 8
    box = M.box_level((4, 4, 8))
    assert box.ncells == 128 and not box.is_cube
    with pytest.raises(ValueError):
        box.ncells_dim
    assert len(M.enumerate_vertex_patches(box)) == 3 * 3 * 7
    assert lvl.cell_multi_index(4095) == (15, 15, 15)


# ----------------------------------------------------------------- config --
def test_smoother_config_validation():
    with pytest.raises(ValueError):
        dg.SmootherConfig(kind="bogus")
    with pytest.raises(ValueError):
        dg.SmootherConfig(omega=0.0)
    with pytest.raises(ValueError):
        dg.SmootherConfig(m_pre=-1)
    with pytest.raises(ValueError):
        dg.SmootherConfig(coloring="x")
    c = dg.SmootherConfig("avs", 0.25)
    assert c.additive and not c.cell_based


def test_make_context_is_host_only_until_used():
    lvl = dg.build_hierarchy(2, 4, 0).levels[0]
    ctx = dg.make_context(lvl, dg.Basis1D.make(3))
    assert ctx.ndofs == 16 * 16 and ctx.layout.grid_shape() == (4, 4, 4, 4)
    assert ctx.layout.global_index(3, (1, 2)) == 3 * 16 + 1 + 2 * 4
    assert ctx._dev is None


def test_module_drivers_check_kind():
    lvl = dg.build_hierarchy(2, 2, 0).levels[0]
    basis = dg.Basis1D.make(1)
    ctx = dg.make_context(lvl, basis)
    s = dg.make_level_smoother(ctx, basis, dg.SmootherConfig("mcs"))
    with pytest.raises(ValueError):
        dg.smooth_additive(s, np.zeros(ctx.ndofs), np.zeros(ctx.ndofs))
    a = dg.make_level_smoother(ctx, basis, dg.SmootherConfig("acs"))
    with pytest.raises(ValueError):
        dg.smooth_multiplicative(a, np.zeros(ctx.ndofs), np.zeros(ctx.ndofs))
    with pytest.raises(NotImplementedError):
        dg.make_level_smoother(ctx, basis, dg.SmootherConfig("acs", coloring="graph"))


# ------------------------------------------------------------- work model --
def test_step_work_matches_survey_table():
    f, b = F.step_work("avs", 3, 3, (32, 32, 32))
    assert f == pytest.approx(1.64e9, rel=5e-3) and b == pytest.approx(50.3e6, rel=5e-3)
    f, b = F.step_work("mvs", 3, 7, (32, 32, 32))
    assert f == pytest.approx(4.27e10, rel=5e-3) and b == pytest.approx(2.93e9, rel=5e-3)
    f, _ = F.step_work("acs", 3, 15, (16, 16, 16))
    assert f == pytest.approx(7.75e9, rel=5e-3)
    f, b = F.step_work("avs", 3, 5, (64, 64, 64))
    assert f == pytest.approx(6.85e10, rel=5e-3) and b == pytest.approx(1.36e9, rel=5e-3)


def test_reference_operator_flop_convention():
    """The reference FlopCounter for one 3D Q3/Q7/Q15 apply at 16^3 cells
    (71 / 848 / 11,145 MFLOP)."""
    for k, want in ((3, 71e6), (7, 848e6), (15, 11145e6)):
        got = F.operator_apply_flops(3, k + 1, k + 1, (16, 16, 16))
        assert got == pytest.approx(want, rel=1e-2)


# --------------------------------------------------- live reference (opt) --
@pytest.mark.skipif(not have_reference(), reason="reference tree not mounted")
def test_host_tables_equal_reference_bitwise():
    sys.path.insert(0, REF_SRC)
    try:
        from dgmg import fastdiag as rfd, mesh as rmesh
        from dgmg.polybasis import Basis1D as RBasis
        for d, nc, k in ((3, 4, 3), (3, 5, 5), (2, 6, 7)):
            lvl = rmesh.build_hierarchy(d, nc, 0).levels[0]
            rb = RBasis.make(k)
            ours = T.build_tables(B.Basis1D.make(k), 1.0 / nc, (nc,) * d)
            cset = rfd.CellSolverSet(lvl, rb, 1.0)
            for ids, solver in cset.classes:
                code = int(cset.class_of[ids[0]])
                want = solver.inv_sum_rev.transpose(tuple(range(d - 1, -1, -1))).ravel()
                assert np.array_equal(ours.cell_invsum[code], want)
            pset = rfd.PatchSolverSet(lvl, rb, 1.0)
            for rows, solver, _ in pset.classes:
                code = int(pset.class_of[rows[0]])
                want = solver.inv_sum_rev.transpose(tuple(range(d - 1, -1, -1))).ravel()
                assert np.array_equal(ours.patch_invsum[code], want)
                for t in range(d):
                    dig = (code >> (2 * t)) & 3
                    assert np.array_equal(np.abs(ours.patch_z[dig]),
                                          np.abs(solver.eigenpairs[t].vectors))
    finally:
        sys.path.remove(REF_SRC)
