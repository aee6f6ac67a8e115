"""GPU parity: the CUDA path through the public API (C ABI underneath)
against the reference's golden vectors and the pinned CPU oracle.

Tolerance (north star): relative L2 <= 1e-12 in fp64; index maps bit-exact.
"""
import os
import numpy as np
import pytest
import torch

from _common import golden, inputs, rel, RTOL

import paper_1910_11239_b200 as dg
from paper_1910_11239_b200 import fastdiag as fd
from paper_1910_11239_b200 import mesh as M
from oracle.sipg_oracle import OracleLevel

pytestmark = pytest.mark.gpu
G = golden()
OPS = sorted({k.split("/")[0] for k in G if k.startswith("op_")})
STEPS = sorted({k.split("/")[0] for k in G if k.startswith("sm_")})


def _experimental():
    from paper_1910_11239_b200 import _lib
    return bool(_lib.load().dg_build_flags() & 1)


experimental = pytest.mark.skipif(not _experimental(), reason="built without -DDGB_EXPERIMENTAL")


def _setup(d, nc, k, kind="acs", omega=1.0):
    lvl = dg.build_hierarchy(d, nc, 0).levels[0]
    basis = dg.Basis1D.make(k)
    ctx = dg.make_context(lvl, basis, 1.0)
    sm = dg.make_level_smoother(ctx, basis, dg.SmootherConfig(kind=kind, omega=omega))
    return ctx, basis, sm


# ---------------------------------------------------------------- operator --
@pytest.mark.parametrize("name", OPS)
def test_operator_and_residual_match_reference(name):
    _, d, k, nc = name.split("_")
    ctx, _, _ = _setup(int(d[0]), int(nc[1:]), int(k[1:]))
    x0, b = inputs(ctx.ndofs)
    v = dg.apply_operator(ctx, x0)
    assert rel(v, G[name + "/Ax"]) <= RTOL
    r = np.empty(ctx.ndofs)
    out = dg.residual(ctx, x0, b, out=r)
    assert out is r and rel(r, G[name + "/res"]) <= RTOL
    # torch zero-copy path gives the same bits as the numpy path
    xt = torch.from_numpy(x0).cuda()
    vt = dg.apply_operator(ctx, xt)
    assert isinstance(vt, torch.Tensor) and np.array_equal(vt.cpu().numpy(), v)


@pytest.mark.parametrize("d,nc,k", [(2, 64, 3), (3, 32, 3), (3, 16, 15), (3, 12, 7),
                                    (3, 16, 5), (2, 9, 9), (3, 5, 11), (3, 7, 6), (3, 6, 4)])
def test_operator_matches_oracle_at_size(d, nc, k):
    ctx, _, _ = _setup(d, nc, k)
    x0, b = inputs(ctx.ndofs, 11)
    lvl = OracleLevel((nc,) * d, k)
    assert rel(dg.apply_operator(ctx, x0), lvl.apply(x0)) <= RTOL
    r = np.empty(ctx.ndofs)
    assert rel(dg.residual(ctx, x0, b, out=r), lvl.residual(x0, b)) <= RTOL


@pytest.mark.parametrize("k", [3, 5, 6, 7, 8, 11, 12, 15])
def test_residual_kernel_variants_agree(k, monkeypatch):
    """res2 (five passes) and res3 (three passes, mass-transformed face
    fields) regroup the same sums: equal to rounding, and both at the oracle."""
    ctx, _, _ = _setup(3, 7, k)
    x0, b = inputs(ctx.ndofs, 12)
    want = OracleLevel((7,) * 3, k).residual(x0, b)
    got = {}
    for v in ("0", "1"):
        monkeypatch.setenv("DGB_RES3", v)
        monkeypatch.setenv("DGB_RES3_HI", v)
        got[v] = dg.residual(ctx, x0, b, out=np.empty(ctx.ndofs))
        assert rel(got[v], want) <= RTOL
    assert rel(got["0"], got["1"]) <= 1e-14


def test_operator_symmetric_full_cfg5_size():
    """Size-independent property at the cfg-5 size (64^3 Q5): u.Av = v.Au."""
    ctx, _, _ = _setup(3, 64, 5)
    u = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1)) - 0.5
    v = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2)) - 0.5
    au = dg.apply_operator(ctx, u)
    av = dg.apply_operator(ctx, v)
    a = float(torch.dot(u, av))
    b = float(torch.dot(v, au))
    assert abs(a - b) <= 1e-12 * float(torch.dot(u, au))
    assert float(torch.dot(u, au)) > 0


def test_operator_errors():
    ctx, _, _ = _setup(2, 3, 2)
    with pytest.raises(ValueError):
        dg.apply_operator(ctx, np.zeros(ctx.ndofs + 1))
    t = torch.zeros(ctx.ndofs, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        dg.apply_operator(ctx, t, out=t)
    with pytest.raises(ValueError):
        dg.residual(ctx, t, t.clone(), out=t)


# --------------------------------------------------------------- smoothing --
@pytest.mark.parametrize("name", STEPS)
def test_smoothing_step_matches_reference(name):
    kind = name.split("_")[1]
    d, nc, k, om, rev = G[name + "/meta"]
    ctx, _, sm = _setup(int(d), int(nc), int(k), kind, float(om))
    x0, b = inputs(ctx.ndofs)
    x = x0.copy()
    sm.smooth(x, b, reverse=bool(rev))
    assert rel(x, G[name + "/x"]) <= RTOL
    assert rel(x - x0, G[name + "/x"] - x0) <= 1e-11


@pytest.mark.parametrize("kind,d,nc,k,omega", [
    ("acs", 2, 64, 3, 0.7),     # cfg 1 (full size)
    ("avs", 3, 32, 3, 0.25),    # cfg 2 (full size)
    ("acs", 3, 16, 15, 0.7),    # cfg 4 (full size)
    ("mvs", 3, 10, 7, 1.0),     # cfg 3 at reduced n_c
    ("avs", 3, 20, 5, 0.25),    # cfg 5 at reduced n_c
    ("mcs", 3, 9, 4, 0.8),
    ("mvs", 2, 17, 6, 1.0),
])
def test_smoothing_step_matches_oracle_at_size(kind, d, nc, k, omega):
    ctx, _, sm = _setup(d, nc, k, kind, omega)
    x0, b = inputs(ctx.ndofs, 3)
    x = torch.from_numpy(x0).cuda()
    sm.smooth(x, torch.from_numpy(b).cuda())
    want = OracleLevel((nc,) * d, k).smooth(kind, omega, x0, b)
    got = x.cpu().numpy()
    assert rel(got, want) <= RTOL
    assert rel(got - x0, want - x0) <= 1e-11


@pytest.mark.parametrize("seed", [0, 1])
def test_full_cfg5_avs_step_matches_oracle(seed):
    """cfg 5 at the size bench.py times it (3D Q5, 64^3 cells, 56.6M DoFs, AVS
    omega 1/4, the default one-launch bulk reduce-add path) against the CPU
    oracle (~30-60 s of host work per seed)."""
    ctx, _, sm = _setup(3, 64, 5, "avs", 0.25)
    x0, b = inputs(ctx.ndofs, seed)
    x = torch.from_numpy(x0).cuda()
    sm.smooth(x, torch.from_numpy(b).cuda())
    got = x.cpu().numpy()
    del x
    want = OracleLevel((64,) * 3, 5).smooth("avs", 0.25, x0, b)
    assert rel(got, want) <= RTOL
    assert rel(got - x0, want - x0) <= 1e-11


def test_full_cfg3_mvs_sweep_matches_oracle():
    """cfg 3 at the size bench.py times it (3D Q7, 32^3 cells, 16.8M DoFs, one
    MVS sweep over 16 colours, omega 1) against the CPU oracle."""
    ctx, _, sm = _setup(3, 32, 7, "mvs", 1.0)
    x0, b = inputs(ctx.ndofs, 0)
    x = torch.from_numpy(x0).cuda()
    sm.smooth(x, torch.from_numpy(b).cuda())
    got = x.cpu().numpy()
    want = OracleLevel((32,) * 3, 7).smooth("mvs", 1.0, x0, b)
    assert rel(got, want) <= RTOL
    assert rel(got - x0, want - x0) <= 1e-11


def test_mvs_full_cfg3_last_colour_local_residuals_vanish():
    """cfg 3 at full size (3D Q7, 32^3, 16 colours, omega=1): after the sweep,
    R_j (b - A x) = 0 on every patch of the last colour (exact local solves)."""
    ctx, _, sm = _setup(3, 32, 7, "mvs", 1.0)
    x0, b = inputs(ctx.ndofs, 0)
    x = torch.from_numpy(x0).cuda()
    bd = torch.from_numpy(b).cuda()
    sm.smooth(x, bd)
    r = torch.empty_like(x)
    dg.residual(ctx, x, bd, out=r)
    last = sm.colors.sets[-1]
    gi = torch.from_numpy(sm.set.gather_map(last)).cuda()
    loc = r[gi]
    assert float(loc.norm()) <= 1e-12 * float(bd.norm())
    assert float(r.norm()) > 1e-3 * float(bd.norm())  # not trivially zero elsewhere


def test_avs_full_cfg5_linear_in_b():
    """cfg 5 at full size (64^3 Q5 AVS): S(x, 2b) - S(x, 0) = 2 (S(x, b) - S(x, 0))."""
    ctx, _, sm = _setup(3, 64, 5, "avs", 0.25)
    x0, b = inputs(ctx.ndofs, 0)
    xd = torch.from_numpy(x0).cuda()
    bd = torch.from_numpy(b).cuda()
    outs = []
    for s in (0.0, 1.0, 2.0):
        x = xd.clone()
        sm.smooth(x, bd * s)
        outs.append(x)
    d1 = outs[1] - outs[0]
    d2 = outs[2] - outs[0]
    assert float((d2 - 2 * d1).norm()) <= 1e-12 * float(d2.norm())


def test_cfg5_host_pipelined_step_matches_device_step():
    """cfg 5 at full size through the e2e path: pinned host tensors take the
    pipelined step (16 z-chunks + 2-layer tail chunks, H2D / residual / range
    solves / D2H overlapped) and give the device-resident step's update to
    rounding (both accumulate the patch updates with bulk fp64 reduce-adds)."""
    ctx, _, sm = _setup(3, 64, 5, "avs", 0.25)
    x0, b = inputs(ctx.ndofs, 0)
    xh = torch.from_numpy(x0.copy()).pin_memory()
    bh = torch.from_numpy(b).pin_memory()
    assert sm._pipelinable(xh, bh)
    bounds = sm._pipe_bounds(64)
    assert bounds[-1] == 64 and bounds[-2] == 62  # the tail chunks are in use
    sm.smooth(xh, bh)
    xd = torch.from_numpy(x0).cuda()
    sm.smooth(xd, bh.cuda())
    want = xd.cpu() - torch.from_numpy(x0)
    got = xh - torch.from_numpy(x0)
    assert float((got - want).norm()) <= 1e-13 * float(want.norm())


def test_graph_and_direct_launch_agree_bitwise():
    ctx, _, sm = _setup(3, 6, 3, "mvs", 1.0)
    x0, b = inputs(ctx.ndofs)
    x1 = x0.copy()
    sm.use_graph = True
    sm.smooth(x1, b)
    x2 = x0.copy()
    sm.use_graph = False
    sm.smooth(x2, b)
    assert np.array_equal(x1, x2)
    x3 = x0.copy()
    sm.use_graph = True
    sm.smooth(x3, b)  # replay
    assert np.array_equal(x1, x3)


def test_colored_equals_uncolored_additive_patches():
    """`test_smoothers.py:74-84` on the device: colour-by-colour writes vs one
    atomic launch over all patches."""
    ctx, _, sm = _setup(2, 8, 2, "avs", 0.2)
    _, b = inputs(ctx.ndofs, 4)
    x1 = np.zeros(ctx.ndofs)
    sm.smooth_additive(x1, b)
    x2 = np.zeros(ctx.ndofs)
    sm.smooth_additive_uncolored(x2, b)
    assert np.allclose(x1, x2, atol=1e-13 * max(1.0, np.abs(x1).max()))
    x3 = np.zeros(ctx.ndofs)
    rev = M.ColorPartition(sm.colors.n_subdomains, sm.colors.sets[::-1])
    sm.smooth_additive(x3, b, colors=rev)
    assert np.allclose(x1, x3, atol=1e-13 * max(1.0, np.abs(x1).max()))


def test_exact_single_cell_and_single_patch_solves():
    for d, nc, k, kind in ((2, 1, 3, "acs"), (2, 2, 2, "avs"), (3, 1, 4, "acs"), (3, 2, 2, "avs")):
        ctx, _, sm = _setup(d, nc, k, kind, 1.0)
        b = np.random.default_rng(0).standard_normal(ctx.ndofs)
        x = np.zeros(ctx.ndofs)
        sm.smooth(x, b)
        r = b - dg.apply_operator(ctx, x)
        assert np.linalg.norm(r) <= 1e-12 * np.linalg.norm(b)


# ------------------------------------------------------------ solver sets --
def test_solver_sets_match_reference():
    lvl = dg.build_hierarchy(3, 4, 0).levels[0]
    basis = dg.Basis1D.make(3)
    ctx = dg.make_context(lvl, basis)
    _, r = inputs(ctx.ndofs, 7)
    cset = fd.CellSolverSet(lvl, basis, 1.0, ctx=ctx)
    x = np.zeros(ctx.ndofs)
    cset.solve_scaled_into(x, r, None, 1.0)
    assert rel(x, G["cellset_3d_q3_n4/x"]) <= RTOL
    x = np.zeros(ctx.ndofs)
    cset.solve_scaled_into(x, r, np.array([0, 5, 21, 63]), 0.5)
    assert rel(x, G["cellset_sub_3d_q3_n4/x"]) <= RTOL
    touched = np.zeros(ctx.ndofs, bool)
    for c in (0, 5, 21, 63):
        touched[c * 64:(c + 1) * 64] = True
    assert np.all(x[~touched] == 0.0)
    pset = fd.PatchSolverSet(lvl, basis, 1.0, ctx=ctx)
    x = np.zeros(ctx.ndofs)
    pset.solve_scaled_into(x, r, None, 1.0, safe_accumulate=True)
    assert rel(x, G["patchset_3d_q3_n4/x"]) <= RTOL
    # reference per-class part format is accepted too
    parts = [np.arange(len(rows)) for rows, _ in pset.classes]
    x2 = np.zeros(ctx.ndofs)
    pset.solve_partitioned(x2, r, parts, 1.0, safe_accumulate=True)
    assert np.allclose(x2, x, rtol=0, atol=1e-13 * np.abs(x).max())


# ------------------------------------------------------------- index maps --
@pytest.mark.parametrize("name", ["map_3d_q3_n4", "map_2d_q2_n5", "map_3d_q1_n5"])
def test_gather_maps_bit_exact(name):
    _, d, k, nc = name.split("_")
    lvl = dg.build_hierarchy(int(d[0]), int(nc[1:]), 0).levels[0]
    basis = dg.Basis1D.make(int(k[1:]))
    pset = fd.PatchSolverSet(lvl, basis, 1.0)
    gi = pset.gather_map(np.arange(len(pset.patches)))
    assert gi.dtype == np.int64 and np.array_equal(gi, G[name + "/gidx"])
    assert np.array_equal(pset.subdomain_indices(3), G[name + "/gidx"][3])


@pytest.mark.parametrize("name,d,nc", [("col_3d_n8", 3, 8), ("col_2d_n7", 2, 7),
                                       ("col_3d_n5", 3, 5)])
def test_device_colour_lists_bit_exact(name, d, nc):
    ctx, _, sm = _setup(d, nc, 1, "mvs", 1.0)
    dev = ctx.dev
    ids = []
    for c in range(dev.num_colours("mvs")):
        ptr, cnt = dev.colour_list("mvs", c)
        ids.append(_read_i32(ptr, cnt))
    assert np.array_equal(np.concatenate(ids), G[name + "/patch_order"])
    rb = [_read_i32(*dev.colour_list("mcs", c)) for c in range(dev.num_colours("mcs"))]
    assert np.array_equal(np.concatenate(rb), G[name + "/rb_order"])


def _read_i32(ptr, cnt):
    """Copy a device int32 array owned by the level to the host."""
    class _View:
        __cuda_array_interface__ = {"shape": (cnt,), "typestr": "<i4",
                                    "data": (ptr, False), "version": 3}
    return torch.as_tensor(_View(), device="cuda").cpu().numpy().copy()


def test_patch_degree_above_templates_is_supported():
    """Degree 8 patches (m = 18) run the generic kernel (csrc/fdmg.cuh); the
    reference has no degree limit (`fastdiag.py:510-634`)."""
    lvl = dg.build_hierarchy(3, 3, 0).levels[0]
    basis = dg.Basis1D.make(8)
    ctx = dg.make_context(lvl, basis)
    sm = dg.make_level_smoother(ctx, basis, dg.SmootherConfig("avs", 0.25))
    assert sm.set.m1 == 18


@experimental
@pytest.mark.parametrize("d,nc,k", [(3, 12, 3), (3, 10, 5), (2, 20, 4), (3, 9, 7)])
def test_dataflow_avs_kernel_bitwise_equals_colour_launches(d, nc, k, monkeypatch):
    """The persistent dataflow AVS kernel (DGB_FLOW=1, flow.cuh) reorders the
    work across z-blocks but keeps every DoF's colour order: bit-identical."""
    ctx, _, sm = _setup(d, nc, k, "avs", 0.25)
    x0, b = inputs(ctx.ndofs, 6)
    monkeypatch.setenv("DGB_CLUSTER", "0")
    monkeypatch.setenv("DGB_AVS_ATOMIC", "0")
    monkeypatch.setenv("DGB_FLOW", "0")
    # the dataflow kernel's residual tasks run res2's arithmetic
    monkeypatch.setenv("DGB_RES3", "0")
    xa = x0.copy()
    sm.smooth(xa, b)
    monkeypatch.setenv("DGB_FLOW", "1")
    assert ctx.dev._lib.dg_flow_enabled(ctx.dev.handle) == 1
    xb = x0.copy()
    sm.use_graph = False
    sm.smooth(xb, b)
    assert np.array_equal(xa, xb)
    want = OracleLevel((nc,) * d, k).smooth("avs", 0.25, x0, b)
    assert rel(xb, want) <= RTOL


@experimental
@pytest.mark.parametrize("d,nc,k", [(3, 12, 3), (3, 9, 5), (2, 21, 4), (3, 7, 7), (3, 2, 2)])
def test_cluster_avs_matches_colour_launches_and_oracle(d, nc, k, monkeypatch):
    """The default additive patch path solves 2^d-patch clusters per launch
    (cluster_kernel): same update, different summation order per DoF."""
    ctx, _, sm = _setup(d, nc, k, "avs", 0.25)
    x0, b = inputs(ctx.ndofs, 8)
    monkeypatch.setenv("DGB_AVS_ATOMIC", "0")
    monkeypatch.setenv("DGB_CLUSTER", "0")
    xa = x0.copy()
    sm.use_graph = False
    sm.smooth(xa, b)
    monkeypatch.setenv("DGB_CLUSTER", "1")
    xb = x0.copy()
    sm.smooth(xb, b)
    assert rel(xb - x0, xa - x0) <= 1e-13
    want = OracleLevel((nc,) * d, k).smooth("avs", 0.25, x0, b)
    assert rel(xb, want) <= RTOL


@pytest.mark.parametrize("d,nc,k", [(3, 12, 3), (2, 21, 4), (3, 5, 7)])
def test_single_launch_atomic_avs_matches_colour_launches(d, nc, k, monkeypatch):
    """Small levels run the additive patch step as one launch with fp64
    reductions (DGB_AVS_ATOMIC); equal to the colour launches up to rounding."""
    ctx, _, sm = _setup(d, nc, k, "avs", 0.25)
    sm.use_graph = False
    x0, b = inputs(ctx.ndofs, 9)
    monkeypatch.setenv("DGB_HOST_PIPELINE", "0")  # numpy inputs: the one-launch device step
    monkeypatch.setenv("DGB_AVS_ATOMIC", "0")
    xa = x0.copy()
    sm.smooth(xa, b)
    monkeypatch.setenv("DGB_AVS_ATOMIC", "1")
    xb = x0.copy()
    sm.smooth(xb, b)
    assert ctx.dev._lib.dg_last_launch_count(ctx.dev.handle) == 2
    assert rel(xb - x0, xa - x0) <= 1e-13


@pytest.mark.parametrize("d,nc,k", [(3, 12, 3), (3, 9, 5), (2, 21, 4), (3, 7, 7)])
def test_parity_class_launches_bitwise_equal_colour_launches(d, nc, k, monkeypatch):
    """The additive step launches colours 2q and 2q+1 together (same vertex
    parity: write-disjoint); every dof keeps its update order, so the result
    is bitwise the 16-colour sequence.  z-windowed class order (DGB_AVS_WIN)
    changes only the order of boundary-layer updates (rounding)."""
    monkeypatch.setenv("DGB_AVS_ATOMIC", "0")
    monkeypatch.setenv("DGB_AVS_COLOURS", "1")
    ctx, _, sm = _setup(d, nc, k, "avs", 0.25)
    x0, b = inputs(ctx.ndofs, 10)
    sm.use_graph = False
    xa = x0.copy()
    sm.smooth(xa, b)
    assert ctx.dev._lib.dg_last_launch_count(ctx.dev.handle) == 1 + 2 ** (d + 1)
    monkeypatch.setenv("DGB_AVS_COLOURS", "0")
    xb = x0.copy()
    sm.smooth(xb, b)
    assert ctx.dev._lib.dg_last_launch_count(ctx.dev.handle) == 1 + 2 ** d
    assert np.array_equal(xa, xb)
    if not _experimental():
        return
    monkeypatch.setenv("DGB_AVS_WIN", "2")
    ctx2, _, sm2 = _setup(d, nc, k, "avs", 0.25)
    xc = x0.copy()
    sm2.smooth(xc, b)
    assert rel(xc - x0, xa - x0) <= 1e-14
    want = OracleLevel((nc,) * d, k).smooth("avs", 0.25, x0, b)
    assert rel(xc, want) <= RTOL


@experimental
@pytest.mark.parametrize("d,nc,k,chunk", [(3, 12, 3, 2), (3, 10, 5, 4), (3, 9, 7, 2)])
def test_overlapped_avs_step_matches_colour_launches(d, nc, k, chunk, monkeypatch):
    """Opt-in overlapped AVS step (DGB_AVS_OVERLAP=1): residual z-chunks on a
    second stream next to the patch-solve chunks, event dependencies keep
    every residual ahead of the updates it reads (rounding-level equal)."""
    monkeypatch.setenv("DGB_AVS_ATOMIC", "0")
    monkeypatch.setenv("DGB_HOST_PIPELINE", "0")  # numpy inputs: the device step
    ctx, _, sm = _setup(d, nc, k, "avs", 0.25)
    x0, b = inputs(ctx.ndofs, 12)
    xa = x0.copy()
    sm.smooth(xa, b)
    monkeypatch.setenv("DGB_AVS_ATOMIC", "1")
    monkeypatch.setenv("DGB_AVS_OVERLAP", "1")
    monkeypatch.setenv("DGB_AVS_CHUNK", str(chunk))
    for lead in ("1", "2"):
        monkeypatch.setenv("DGB_AVS_LEAD", lead)
        ctx2, _, sm2 = _setup(d, nc, k, "avs", 0.25)
        sm2.use_graph = lead == "1"
        xb = x0.copy()
        sm2.smooth(xb, b)
        assert ctx2.dev._lib.dg_last_launch_count(ctx2.dev.handle) > 2
        assert rel(xb - x0, xa - x0) <= 1e-14


@pytest.mark.parametrize("kind,omega,k", [("avs", 0.25, 3), ("acs", 0.7, 3), ("avs", 0.25, 5)])
def test_host_pipelined_step_matches_device_step(kind, omega, k):
    """Host vectors (numpy, pinned tensors) take the pipelined path: chunked
    H2D / residual / range solves / D2H; equal to the device-resident step
    (ACS bitwise, AVS to rounding: one-launch AVS accumulates atomically)."""
    nc = 24
    ctx, _, sm = _setup(3, nc, k, kind, omega)
    x0, b = inputs(ctx.ndofs, 13)
    assert sm._pipelinable(x0, b)
    xd = torch.from_numpy(x0).cuda()
    sm.smooth(xd, torch.from_numpy(b).cuda())
    want = xd.cpu().numpy()
    xn = x0.copy()
    sm.smooth(xn, b)
    xt = torch.from_numpy(x0.copy()).pin_memory()
    sm.smooth(xt, torch.from_numpy(b).pin_memory())
    for got in (xn, xt.numpy()):
        if kind == "acs":
            assert np.array_equal(got, want)
        else:
            assert rel(got - x0, want - x0) <= 1e-14
    assert rel(xn, OracleLevel((nc,) * 3, k).smooth(kind, omega, x0, b)) <= RTOL


@pytest.mark.parametrize("kind,omega", [("acs", 0.7), ("avs", 0.25)])
@pytest.mark.parametrize("head,tail,layers,nc", [(4, 4, 4, 24), (2, 6, 6, 24), (0, 8, 2, 24),
                                                  (0, 4, 4, 13), (0, 4, 4, 17)])
def test_host_pipelined_uneven_chunks(kind, omega, head, tail, layers, nc, monkeypatch):
    """2-layer head / tail chunks around the uniform ones (DGB_PIPE_HEAD /
    DGB_PIPE_TAIL / DGB_PIPE_LAYERS): same result as the device step.  Odd
    nz (13, 17) would leave a 1-layer chunk before the tail, which the
    bounds merge away."""
    monkeypatch.setenv("DGB_PIPE_HEAD", str(head))
    monkeypatch.setenv("DGB_PIPE_TAIL", str(tail))
    monkeypatch.setenv("DGB_PIPE_LAYERS", str(layers))
    ctx, _, sm = _setup(3, nc, 2, kind, omega)
    bounds = sm._pipe_bounds(nc)
    assert bounds[0] == 0 and bounds[-1] == nc and all(b - a >= 2 for a, b in zip(bounds, bounds[1:]))
    x0, b = inputs(ctx.ndofs, 15)
    assert sm._pipelinable(x0, b)
    xd = torch.from_numpy(x0).cuda()
    sm.smooth(xd, torch.from_numpy(b).cuda())
    want = xd.cpu().numpy()
    xn = x0.copy()
    sm.smooth(xn, b)
    if kind == "acs":
        assert np.array_equal(xn, want)
    else:
        assert rel(xn - x0, want - x0) <= 1e-14


@pytest.mark.parametrize("k", [3, 5])
def test_mvs_block_list_residual_bitwise(k, monkeypatch):
    """The MVS restricted residual on vertex-patch cell lists runs in 2x2x2
    block mode (in-block neighbour traces from shared memory): bitwise the
    per-cell list mode, and at the oracle."""
    ctx, _, sm = _setup(3, 6, k, "mvs", 1.0)
    x0, b = inputs(ctx.ndofs, 14)
    out = {}
    for v in ("0", "1"):
        monkeypatch.setenv("DGB_RES_BLOCK_LIST", v)
        sm.use_graph = False
        x = x0.copy()
        sm.smooth(x, b)
        out[v] = x
    assert np.array_equal(out["0"], out["1"])
    want = OracleLevel((6,) * 3, k).smooth("mvs", 1.0, x0, b)
    assert rel(out["1"], want) <= RTOL


def test_local_solver_apply_inverse_is_exact_local_solve():
    """`LocalSolver.apply_inverse` (fastdiag.py:118-133) on the device: the
    cell solver inverts the Kronecker-sum cell matrix, the patch solver the
    dense patch restriction of the operator (oracle dense matrix)."""
    lvl = dg.build_hierarchy(3, 3, 0).levels[0]
    basis = dg.Basis1D.make(2)
    ctx = dg.make_context(lvl, basis)
    ol = OracleLevel((3, 3, 3), 2)
    a = ol.dense()
    rng = np.random.default_rng(12)
    cset = fd.CellSolverSet(lvl, basis, 1.0, ctx=ctx)
    for cell in (0, 13, 26):
        solver = cset.local_solver(cell)
        idx = np.arange(cell * 27, (cell + 1) * 27)
        r = rng.standard_normal(27)
        want = np.linalg.solve(a[np.ix_(idx, idx)], r)
        assert rel(solver.apply_inverse(r), want) <= 1e-12
        assert rel(fd.apply_inverse(solver, r.reshape(3, 3, 3)).ravel(), want) <= 1e-12
    pset = fd.PatchSolverSet(lvl, basis, 1.0, ctx=ctx)
    for j in range(len(pset.patches)):
        idx = pset.subdomain_indices(j)
        r = rng.standard_normal(idx.size)
        want = np.linalg.solve(a[np.ix_(idx, idx)], r)
        assert rel(pset.local_solver(j).apply_inverse(r), want) <= 1e-12
    with pytest.raises(ValueError):
        cset.local_solver(0).apply_inverse(np.zeros(5))


def test_numpy_views_update_in_place_and_readonly_raises():
    """x may be a non-contiguous numpy view (updated in place, like the
    reference's in-place numpy arithmetic); a read-only x raises instead of
    silently dropping the update."""
    ctx, _, sm = _setup(3, 3, 2, "mvs", 1.0)
    x0, b = inputs(ctx.ndofs, 21)
    want = x0.copy()
    sm.smooth(want, b)
    big = np.zeros(2 * ctx.ndofs)
    view = big[::2]
    view[:] = x0
    sm.smooth(view, b)
    assert np.array_equal(big[::2], want) and not big[1::2].any()
    ro = x0.copy()
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        sm.smooth(ro, b)


def test_library_build_flags():
    """The default library has neither the experimental variants nor the
    bounds checks compiled in; a DGB_LIB build reports what it carries."""
    from paper_1910_11239_b200 import _lib
    flags = _lib.load().dg_build_flags()
    if os.environ.get("DGB_LIB"):
        assert flags >= 0
    else:
        assert flags == 0


@pytest.mark.parametrize("k,nc,rev", [(3, 16, False), (7, 16, True), (2, 17, False)])
def test_mvs_host_wavefront_pipeline_bitwise(k, nc, rev, monkeypatch):
    """Host vectors take the wavefront-pipelined MVS sweep (dg_mvs_range per
    colour and z-chunk, copies overlapped): bitwise the device sweep, for
    numpy (eager) and pinned tensors (one CUDA graph), forward and reverse."""
    monkeypatch.setenv("DGB_MVS_PIPELINE", "1")
    ctx, _, sm = _setup(3, nc, k, "mvs", 1.0)
    x0, b = inputs(ctx.ndofs, 17)
    assert sm._mvs_pipelinable(x0, b)
    xd = torch.from_numpy(x0).cuda()
    sm.smooth(xd, torch.from_numpy(b).cuda(), reverse=rev)
    want = xd.cpu().numpy()
    xn = x0.copy()
    sm.smooth(xn, b, reverse=rev)
    assert np.array_equal(xn, want)
    xh = torch.from_numpy(x0.copy()).pin_memory()
    bh = torch.from_numpy(b).pin_memory()
    for _ in range(2):  # capture, then replay
        xh.copy_(torch.from_numpy(x0))
        sm.smooth(xh, bh, reverse=rev)
        assert np.array_equal(xh.numpy(), want)


def test_recurring_numpy_buffers_are_page_locked_in_place(monkeypatch):
    """The same numpy arrays passed a second time are registered in place
    (cudaHostRegister): results are unchanged, the later calls take the pinned
    pipeline, and the registration goes away with the array."""
    import gc
    from paper_1910_11239_b200 import _device
    monkeypatch.setattr(_device, "_PIN_MODE", "auto")
    monkeypatch.setattr(_device, "_PIN_MIN_BYTES", 1 << 16)
    ctx, _, sm = _setup(3, 12, 3, "avs", 0.25)
    x0, b = inputs(ctx.ndofs, 5)
    want = x0.copy()
    xd = torch.from_numpy(x0).cuda()
    sm.smooth(xd, torch.from_numpy(b).cuda())
    want = xd.cpu().numpy()
    x = x0.copy()
    ptr = x.ctypes.data
    sm.smooth(x, b)                         # first sighting: pageable
    assert ptr not in _device._pin_live
    assert rel(x, want) <= 1e-14
    x[:] = x0
    sm.smooth(x, b)                         # second sighting: registered
    assert _device._pin_live.get(ptr) == x.nbytes
    assert torch.from_numpy(x).is_pinned()
    assert rel(x, want) <= 1e-14
    x[:] = x0
    sm.smooth(x, b)
    assert rel(x, want) <= 1e-14
    v = x[: ctx.ndofs // 2]                  # a view does not own the memory
    del v
    del x
    gc.collect()
    assert ptr not in _device._pin_live
    # read-only and small arrays are left alone
    ro = b.copy()
    ro.flags.writeable = False
    assert not _device.maybe_pin(ro) and not _device.maybe_pin(ro)
    assert not _device.maybe_pin(np.zeros(8)) and not _device.maybe_pin(np.zeros(8))


@experimental
@pytest.mark.parametrize("k,nc,kind", [(7, 6, "mvs"), (15, 3, "acs"), (5, 6, "avs"), (7, 5, "acs")])
def test_res3_load_variants_bitwise(k, nc, kind, monkeypatch):
    """res3b (batched neighbour-fiber loads) and res3c (TMA-staged rows, pair
    mode on patch-cell lists) keep res3's arithmetic: bitwise equal residuals
    and smoothing steps (the variants are opt-in: measured no faster)."""
    monkeypatch.setenv("DGB_RES3_LO", "1")     # n = 6 on res3 too
    monkeypatch.setenv("DGB_HOST_PIPELINE", "0")
    got = {}
    for name, env in (("res3", {}), ("res3b", {"DGB_RES3_BATCH": "1"}),
                      ("res3c", {"DGB_RES3_TMA": "1"})):
        for kk in ("DGB_RES3_BATCH", "DGB_RES3_TMA"):
            monkeypatch.delenv(kk, raising=False)
        for kk, v in env.items():
            monkeypatch.setenv(kk, v)
        ctx, _, sm = _setup(3, nc, k, kind, 0.25 if kind == "avs" else 1.0)
        x0, b = inputs(ctx.ndofs, 9)
        r = dg.residual(ctx, x0, b, out=np.empty(ctx.ndofs))
        x = x0.copy()
        sm.use_graph = False
        sm.smooth(x, b)
        got[name] = (r, x)
    for name in ("res3b", "res3c"):
        assert np.array_equal(got[name][0], got["res3"][0])
        if kind != "avs":   # the default AVS path sums its updates in arbitrary order
            assert np.array_equal(got[name][1], got["res3"][1])
        else:
            assert rel(got[name][1], got["res3"][1]) <= 1e-14


@experimental
def test_two_fiber_patch_solve_matches_default(monkeypatch):
    """fdm7 (two fibers per thread, opt-in) against the default bulk solve on
    the cfg-5 discretisation, colour by colour (deterministic order): bitwise."""
    monkeypatch.setenv("DGB_AVS_ATOMIC", "0")
    monkeypatch.setenv("DGB_HOST_PIPELINE", "0")
    out = {}
    for v in ("0", "1", "2"):
        monkeypatch.setenv("DGB_FDM7", v)
        ctx, _, sm = _setup(3, 7, 5, "avs", 0.25)
        x0, b = inputs(ctx.ndofs, 4)
        x = x0.copy()
        sm.use_graph = False
        sm.smooth(x, b)
        out[v] = x
    assert np.array_equal(out["1"], out["0"]) and np.array_equal(out["2"], out["0"])


@experimental
@pytest.mark.parametrize("nc,rev", [(2, False), (5, False), (4, True)])
def test_fused_mvs_colour_kernel_bitwise(nc, rev, monkeypatch):
    """mvs_fused_kernel (restricted residual + patch solve per patch, opt-in)
    against the two-launch sweep on 3D Q7: bitwise, and the oracle at 1e-12."""
    monkeypatch.setenv("DGB_HOST_PIPELINE", "0")
    out = {}
    for v in ("0", "1"):
        monkeypatch.setenv("DGB_MVS_FUSED", v)
        ctx, _, sm = _setup(3, nc, 7, "mvs", 1.0)
        x0, b = inputs(ctx.ndofs, 2)
        x = x0.copy()
        sm.use_graph = False
        sm.smooth(x, b, reverse=rev)
        out[v] = x
    assert np.array_equal(out["0"], out["1"])
    want = OracleLevel((nc,) * 3, 7).smooth("mvs", 1.0, x0, b, reverse=rev)
    assert rel(out["1"], want) <= RTOL
