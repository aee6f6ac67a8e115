"""GPU parity of the slab decomposition with P ranks emulated in one process
on one GPU (no kernel waits on another rank: the ghost exchange between the
emulated ranks is a plain device copy, the compute is each rank's own
windowed `dg_smooth`).  The owned DoFs must equal the single-GPU step on the
same box bit for bit (same colours, same per-DoF update order), and the
oracle to 1e-12."""
import numpy as np
import pytest
import torch

from _common import inputs, rel

import paper_1910_11239_b200 as dg
from paper_1910_11239_b200.distributed import SlabLayout, SlabSmoother
from oracle.sipg_oracle import OracleLevel

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["0", "1"], ids=["colour-order", "one-launch-default"])
def avs_atomic(request, monkeypatch):
    """"0": the write-disjoint parity-class launches (deterministic, bitwise
    the single-GPU step); "1" (the default, what bench.py runs): one launch
    over every patch of the window with bulk fp64 reduce-adds (overlaps
    summed in arbitrary order: equal to rounding)."""
    monkeypatch.setenv("DGB_AVS_ATOMIC", request.param)
    return request.param == "1"


def _check_single(got, single, x0, atomic):
    if atomic:
        assert rel(got - x0, single - x0) <= 1e-14
    else:
        assert np.array_equal(got, single)


def _exchange(sms, attr="x"):
    for r, sm in enumerate(sms):
        for peer, _, recv in sm.layout.halo_plan():
            src = [s for (pp, s, _) in sms[peer].layout.halo_plan() if pp == r][0]
            getattr(sm, attr)[recv].copy_(getattr(sms[peer], attr)[src])


def _slab_run(dims, k, kind, omega, world, steps, x0, b):
    sms = [SlabSmoother(dims, k, kind, omega, rank=r, world=world, device="cuda")
           for r in range(world)]
    for sm in sms:
        lay = sm.layout
        w0 = lay.window[0] * lay.layer_dofs
        own = sm.owned
        sm.x[own].copy_(torch.from_numpy(x0[w0 + own.start:w0 + own.stop]))
        sm.b[own].copy_(torch.from_numpy(b[w0 + own.start:w0 + own.stop]))
    _exchange(sms, "b")
    for _ in range(steps):
        _exchange(sms, "x")
        for sm in sms:
            sm._local()
    torch.cuda.synchronize()
    out = np.empty_like(x0)
    for sm in sms:
        lay = sm.layout
        w0 = lay.window[0] * lay.layer_dofs
        own = sm.owned
        out[w0 + own.start:w0 + own.stop] = sm.owned_x().cpu().numpy()
    return out


def _single_run(dims, k, kind, omega, steps, x0, b):
    lvl = dg.box_level(dims)
    basis = dg.Basis1D.make(k)
    ctx = dg.make_context(lvl, basis)
    sm = dg.make_level_smoother(ctx, basis, dg.SmootherConfig(kind=kind, omega=omega))
    x = torch.from_numpy(x0).cuda()
    bd = torch.from_numpy(b).cuda()
    for _ in range(steps):
        sm.smooth(x, bd)
    return x.cpu().numpy()


@pytest.mark.parametrize("dims,k,kind,world,steps", [
    ((6, 5, 8), 2, "avs", 2, 2),
    ((6, 5, 8), 2, "avs", 4, 1),
    ((8, 8, 12), 5, "avs", 3, 2),
    ((5, 6, 8), 3, "acs", 4, 2),
    ((7, 4, 16), 1, "avs", 8, 1),
    ((3, 2, 8), 8, "avs", 2, 1),   # degree-8 patches: the generic kernel on windowed levels
    ((2, 3, 12), 9, "avs", 3, 2),
])
def test_emulated_slabs_equal_single_gpu_and_oracle(dims, k, kind, world, steps, avs_atomic):
    omega = 0.25 if kind == "avs" else 0.7
    n = int(np.prod(dims)) * (k + 1) ** 3
    x0, b = inputs(n, 2)
    got = _slab_run(dims, k, kind, omega, world, steps, x0, b)
    single = _single_run(dims, k, kind, omega, steps, x0, b)
    _check_single(got, single, x0, avs_atomic and kind == "avs")
    want = x0
    lvl = OracleLevel(dims, k, h=1.0 / dims[0])
    for _ in range(steps):
        want = lvl.smooth(kind, omega, want, b)
    assert rel(got, want) <= 1e-12


@pytest.mark.parametrize("world", [2, 4, 8])
def test_emulated_slabs_q5_default_path(world, avs_atomic):
    """The cfg-5 discretisation (3D Q5 AVS, omega 1/4) on a 12x10x32 box in
    P = 2, 4, 8 slabs (16 / 8 / 4 owned layers), both launch orders."""
    dims, k = (12, 10, 32), 5
    n = int(np.prod(dims)) * 216
    x0, b = inputs(n, 6)
    got = _slab_run(dims, k, "avs", 0.25, world, 1, x0, b)
    single = _single_run(dims, k, "avs", 0.25, 1, x0, b)
    _check_single(got, single, x0, avs_atomic)
    want = OracleLevel(dims, k, h=1.0 / dims[0]).smooth("avs", 0.25, x0, b)
    assert rel(got, want) <= 1e-12


def test_cfg5_slab_window_interface_patches(avs_atomic):
    """cfg-5 geometry at P=2 with a reduced 16x16 face (64 layers per rank):
    the rank-1 window starts two layers below its first owned layer and the
    interface patches (v_z = 64) are computed on both ranks."""
    dims, k, world = (16, 16, 128), 5, 2
    lay = SlabLayout(dims, k, 1, world)
    assert lay.window == (62, 128) and lay.pv == (64, 127)
    n = int(np.prod(dims)) * 216
    x0, b = inputs(n, 4)
    got = _slab_run(dims, k, "avs", 0.25, world, 1, x0, b)
    single = _single_run(dims, k, "avs", 0.25, 1, x0, b)
    _check_single(got, single, x0, avs_atomic)


@pytest.mark.parametrize("kind,world", [("avs", 2), ("avs", 3), ("acs", 2)])
def test_split_step_equals_plain_step(kind, world):
    """The halo-overlapped step (interior residual + solves while the halo is
    in flight, then the boundary part; SlabSmoother.split_ranges) computes the
    plain local step: equal to rounding (reduce-add order) on every rank,
    and the oracle to 1e-12."""
    dims, k = (6, 5, 8 * world), 2
    omega = 0.25 if kind == "avs" else 0.7
    n = int(np.prod(dims)) * (k + 1) ** 3
    x0, b = inputs(n, 13)
    plain = _slab_run(dims, k, kind, omega, world, 1, x0, b)
    sms = [SlabSmoother(dims, k, kind, omega, rank=r, world=world, device="cuda")
           for r in range(world)]
    for sm in sms:
        lay = sm.layout
        w0 = lay.window[0] * lay.layer_dofs
        own = sm.owned
        sm.x[own].copy_(torch.from_numpy(x0[w0 + own.start:w0 + own.stop]))
        sm.b[own].copy_(torch.from_numpy(b[w0 + own.start:w0 + own.stop]))
    _exchange(sms, "b")
    # interior before the exchange (it must not need the ghosts), boundary after
    for sm in sms:
        sm._split_part("interior")
    _exchange(sms, "x")
    for sm in sms:
        sm._split_part("boundary")
    torch.cuda.synchronize()
    got = np.empty_like(x0)
    for sm in sms:
        lay = sm.layout
        w0 = lay.window[0] * lay.layer_dofs
        own = sm.owned
        got[w0 + own.start:w0 + own.stop] = sm.owned_x().cpu().numpy()
    assert rel(got - x0, plain - x0) <= 1e-14
    want = OracleLevel(dims, k, h=1.0 / dims[0]).smooth(kind, omega, x0, b)
    assert rel(got, want) <= 1e-12
