"""Multi-process (gloo, world_size 2 and 3) tests of the slab decomposition's
host logic on CPU: layouts, ghost exchange and owned-DoF assembly.

The local compute is injected: it embeds the rank's window into a global
zero vector and runs the oracle's residual and patch/cell solves restricted
to the window's ranges, exactly the work the device `dg_smooth` does on a
windowed level.  If the exchange or the ranges were wrong, the assembled
result would differ from the single-process global step.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _common import inputs, rel

from paper_1910_11239_b200.distributed import SlabLayout, SlabSmoother
from oracle.sipg_oracle import OracleLevel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _window_compute(dims, k, kind, omega, layout):
    """Oracle-backed local step on the rank's window (test-only)."""
    lvl = OracleLevel(dims, k, h=1.0 / dims[0])
    w0, w1 = layout.window
    lo = w0 * layout.layer_dofs
    hi = w1 * layout.layer_dofs

    def compute(x, b, r):
        xg = np.zeros(lvl.ndofs)
        bg = np.zeros(lvl.ndofs)
        xg[lo:hi] = x.numpy()
        bg[lo:hi] = b.numpy()
        rg = lvl.residual(xg, bg)
        r0, r1 = layout.res
        mask = np.zeros(lvl.ndofs, bool)
        mask[r0 * layout.layer_dofs:r1 * layout.layer_dofs] = True
        rg[~mask] = np.nan  # only the residual layers may be read
        if kind == "avs":
            v = lvl.patch_vertices()
            p0, p1 = layout.pv
            ids = np.nonzero((v[:, -1] >= p0) & (v[:, -1] <= p1))[0]
            lvl.patch_solve(xg, rg, omega, ids, safe=True)
        else:
            z0, z1 = layout.own
            cells = np.arange(z0 * layout.layer_dofs // lvl.n ** lvl.d,
                              z1 * layout.layer_dofs // lvl.n ** lvl.d)
            lvl.cell_solve(xg, rg, omega, cells)
        x.copy_(torch.from_numpy(xg[lo:hi]))
    return compute


def _worker(rank, world, port, dims, k, kind, omega, steps, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = SlabLayout(dims, k, rank, world)
        sm = SlabSmoother(dims, k, kind, omega, rank=rank, world=world, device="cpu",
                          compute=_window_compute(dims, k, kind, omega, lay))
        n_glob = int(np.prod(dims)) * (k + 1) ** len(dims)
        x0, b = inputs(n_glob, 3)
        own = slice(lay.layer_slice(*lay.own).start + lay.window[0] * lay.layer_dofs,
                    lay.layer_slice(*lay.own).stop + lay.window[0] * lay.layer_dofs)
        sm.load(x0[own], b[own])
        # ghosts hold the neighbours' data after load()
        w0, w1 = lay.window
        assert np.array_equal(sm.x.numpy(), x0[w0 * lay.layer_dofs:w1 * lay.layer_dofs])
        for _ in range(steps):
            sm.step()
        out_q.put((rank, own.start, sm.owned_x().numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims,k,kind,steps", [
    (2, (3, 3, 8), 1, "avs", 2),
    (3, (3, 2, 9), 2, "avs", 1),
    (2, (4, 3, 6), 1, "acs", 2),
    (4, (3, 3, 8), 1, "avs", 1),
])
def test_slab_step_equals_global_step(world, dims, k, kind, steps):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    omega = 0.25 if kind == "avs" else 0.7
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, k, kind, omega, steps, q))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lvl = OracleLevel(dims, k, h=1.0 / dims[0])
    x0, b = inputs(lvl.ndofs, 3)
    want = x0
    for _ in range(steps):
        want = lvl.smooth(kind, omega, want, b)
    got = np.empty(lvl.ndofs)
    for _, start, xs in parts:
        got[start:start + len(xs)] = xs
    assert rel(got, want) <= 1e-13


def test_slab_layout_ranges():
    lay = SlabLayout((64, 64, 512), 5, 3, 8)
    assert lay.own == (192, 256)
    assert lay.window == (190, 258)
    assert lay.res == (191, 257)
    assert lay.pv == (192, 256)
    assert lay.layer_dofs == 64 * 64 * 216
    plan = lay.halo_plan()
    assert [p[0] for p in plan] == [2, 4]
    first = SlabLayout((64, 64, 512), 5, 0, 8)
    assert first.window == (0, 66) and first.res == (0, 65) and first.pv == (1, 64)
    last = SlabLayout((64, 64, 512), 5, 7, 8)
    assert last.window == (446, 512) and last.pv == (448, 511)
    uneven = [SlabLayout((4, 4, 10), 1, r, 3).own for r in range(3)]
    assert uneven == [(0, 4), (4, 7), (7, 10)]
    with pytest.raises(ValueError):
        SlabLayout((4, 4, 3), 1, 1, 2).validate()


@pytest.mark.parametrize("nz,world,kind", [(24, 2, "avs"), (24, 3, "acs"), (40, 4, "avs"), (18, 3, "avs")])
def test_split_ranges_cover_the_plain_step(nz, world, kind):
    """SlabSmoother.split_ranges: interior + boundary residual layers = the
    residual range, patch (or cell) ranges = the plain step's, and the
    interior part reads no ghost layer and writes no layer a boundary
    residual reads."""
    for rank in range(world):
        sm = SlabSmoother((4, 4, nz), 2, kind, 0.25 if kind == "avs" else 0.7, rank=rank,
                          world=world, device="cpu", compute=lambda *a: None)
        lay = sm.layout
        z0, z1 = lay.own
        rg = sm.split_ranges()
        res = sorted([rg["res_inner"]] + rg["res_outer"])
        cover = set()
        for lo, hi in res:
            cover |= set(range(lo, hi))
        assert cover == set(range(*lay.res))
        sol = sorted([rg["solve_inner"]] + rg["solve_outer"])
        cover = set()
        for lo, hi in sol:
            assert not cover & set(range(lo, hi))
            cover |= set(range(lo, hi))
        want = set(range(lay.pv[0], lay.pv[1] + 1)) if kind == "avs" else set(range(z0, z1))
        assert cover == want
        # interior residual reads x on [lo-1, hi+1): owned layers only
        lo, hi = rg["res_inner"]
        assert lo - 1 >= z0 and hi + 1 <= z1
        # interior writes vs boundary residual reads
        slo, shi = rg["solve_inner"]
        written = set(range(slo - 1, shi)) if kind == "avs" else set(range(slo, shi))
        for blo, bhi in rg["res_outer"]:
            assert not written & set(range(blo - 1, bhi + 1))
        # interior solves read r only where the interior residual wrote it
        read = set(range(slo - 1, shi)) if kind == "avs" else set(range(slo, shi))
        assert read <= set(range(lo, hi))
