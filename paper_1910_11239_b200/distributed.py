"""Slab domain decomposition across the GPUs of one box.

The reference is single-process (`smoothers.py`, no MPI); this is the new
multi-GPU layer of the north star.  A box of nx x ny x nz cells is split into
contiguous slabs of cell layers along the last direction; cell ids (and
therefore DoFs) of a slab are one contiguous range of the canonical vector
(`mesh.py:105-112`, `dgop.py:70-103`).

Per rank with owned layers [z0, z1):

- storage window [z0-2, z1+2) (clipped at the physical boundary): two ghost
  layers of x per side, refreshed every step by NCCL send/recv of the
  neighbours' first/last two owned layers (contiguous memory, no packing);
- residual on [z0-1, z1+1): owned plus the first ghost layer, which needs the
  second ghost layer's face traces;
- every patch whose vertex v_z lies in [z0, z1] (all patches touching an
  owned cell, interface patches computed redundantly by both neighbours);
- writes land on owned layers (and on ghost layers, which the next exchange
  overwrites).

Colours are global, so each owned DoF receives the same updates in the same
order as on one GPU: the slab step is the global AVS/ACS step restricted to
the owned DoFs, bit for bit.  No collective is needed inside the step; the
exchange is a point-to-point halo (`batch_isend_irecv`, NCCL over NVLink on
GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch
import torch.distributed as dist

GHOST = 2


@dataclass(frozen=True)
class SlabLayout:
    """Index bookkeeping of one rank's slab (pure host logic)."""

    dims: tuple
    degree: int
    rank: int
    world: int

    @property
    def d(self) -> int:
        return len(self.dims)

    @property
    def nz(self) -> int:
        return self.dims[-1]

    @property
    def layer_dofs(self) -> int:
        cells = int(np.prod(self.dims[:-1]))
        return cells * (self.degree + 1) ** self.d

    @property
    def own(self) -> tuple:
        base, extra = divmod(self.nz, self.world)
        z0 = self.rank * base + min(self.rank, extra)
        return z0, z0 + base + (1 if self.rank < extra else 0)

    @property
    def window(self) -> tuple:
        z0, z1 = self.own
        return max(0, z0 - GHOST), min(self.nz, z1 + GHOST)

    @property
    def res(self) -> tuple:
        z0, z1 = self.own
        return max(0, z0 - 1), min(self.nz, z1 + 1)

    @property
    def pv(self) -> tuple:
        z0, z1 = self.own
        return max(1, z0), min(self.nz - 1, z1)

    @property
    def n_window(self) -> int:
        w0, w1 = self.window
        return (w1 - w0) * self.layer_dofs

    @property
    def n_owned(self) -> int:
        z0, z1 = self.own
        return (z1 - z0) * self.layer_dofs

    def layer_slice(self, z_lo: int, z_hi: int) -> slice:
        """Local-vector slice of global layers [z_lo, z_hi)."""
        w0, _ = self.window
        return slice((z_lo - w0) * self.layer_dofs, (z_hi - w0) * self.layer_dofs)

    def halo_plan(self):
        """[(peer, send_slice, recv_slice)] for the ghost exchange."""
        z0, z1 = self.own
        plan = []
        if self.rank > 0:
            g = min(GHOST, z0)
            plan.append((self.rank - 1, self.layer_slice(z0, z0 + g), self.layer_slice(z0 - g, z0)))
        if self.rank < self.world - 1:
            g = min(GHOST, self.nz - z1)
            plan.append((self.rank + 1, self.layer_slice(z1 - g, z1), self.layer_slice(z1, z1 + g)))
        return plan

    def validate(self) -> None:
        z0, z1 = self.own
        if z1 - z0 < GHOST and self.world > 1:
            raise ValueError(f"each rank needs >= {GHOST} owned cell layers (got {z1 - z0})")


def halo_exchange(vec: torch.Tensor, layout: SlabLayout, group=None) -> None:
    """Refresh the ghost layers of `vec` from the neighbouring ranks."""
    plan = layout.halo_plan()
    if not plan:
        return
    ops = []
    for peer, send, recv in plan:
        ops.append(dist.P2POp(dist.isend, vec[send], peer, group))
        ops.append(dist.P2POp(dist.irecv, vec[recv], peer, group))
    try:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    except RuntimeError as e:  # NCCL / gloo timeout or a dead peer: say which exchange failed
        peers = sorted({peer for peer, _, _ in plan})
        raise RuntimeError(f"halo exchange of rank {layout.rank} with rank(s) {peers} failed "
                           f"({sum(vec[s].numel() for _, s, _ in plan) * 8} bytes sent): {e}") from e


class SlabSmoother:
    """One rank's part of the multi-GPU AVS/ACS step on a box level.

    `compute(x_local, b_local, r_local)` runs the local step on the window;
    by default it is the device `dg_smooth` on a windowed level.  (The CPU
    tests inject an oracle-backed compute to check the host logic with gloo.)
    """

    def __init__(self, dims, k: int, kind: str = "avs", omega: float = 0.25,
                 rank: int | None = None, world: int | None = None, h: float | None = None,
                 gamma_hat: float = 1.0, device=None,
                 compute: Callable | None = None, group=None):
        if kind not in ("avs", "acs"):
            raise ValueError("multi-GPU slabs support the additive smoothers (avs, acs)")
        rank = dist.get_rank() if rank is None else rank
        world = dist.get_world_size() if world is None else world
        self.layout = SlabLayout(tuple(int(v) for v in dims), int(k), rank, world)
        self.layout.validate()
        self.kind, self.omega, self.group = kind, float(omega), group
        self.h = 1.0 / dims[0] if h is None else h
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None \
            else torch.device(device)
        self._compute = compute
        self._dev = None
        if compute is None:
            self._dev = self._make_device_level(gamma_hat)
        n = self.layout.n_window
        self.x = torch.zeros(n, dtype=torch.float64, device=self.device)
        self.b = torch.zeros(n, dtype=torch.float64, device=self.device)
        self.r = torch.zeros(n, dtype=torch.float64, device=self.device)

    def _make_device_level(self, gamma_hat):
        from . import _lib
        from .basis import Basis1D
        from .tables import build_tables

        lay = self.layout
        tables = build_tables(Basis1D.make(lay.degree), self.h, lay.dims, gamma_hat,
                              with_patches=self.kind == "avs")
        w0, w1 = lay.window
        return _lib.DeviceLevel(tables, lay.dims, z_begin=w0, z_count=w1 - w0, own=lay.own,
                                res=lay.res, pv=lay.pv)

    @property
    def n_owned(self) -> int:
        return self.layout.n_owned

    @property
    def owned(self) -> slice:
        return self.layout.layer_slice(*self.layout.own)

    def load(self, x_owned, b_owned) -> None:
        """Copy this rank's owned parts of x and b in, fill the ghosts."""
        self.x[self.owned].copy_(torch.as_tensor(np.asarray(x_owned)).to(self.device))
        self.b[self.owned].copy_(torch.as_tensor(np.asarray(b_owned)).to(self.device))
        halo_exchange(self.b, self.layout, self.group)
        halo_exchange(self.x, self.layout, self.group)

    def _local(self) -> None:
        if self._compute is not None:
            self._compute(self.x, self.b, self.r)
            return
        from . import _lib
        from ._device import stream_handle

        dev = self._dev
        _lib.check(dev._lib.dg_smooth(dev.handle, _lib.KINDS[self.kind], self.omega, 0,
                                      self.x.data_ptr(), self.b.data_ptr(), self.r.data_ptr(),
                                      1, stream_handle()))

    def step(self) -> None:
        """Ghost exchange and the local additive step (one per smoothing step).
        On the device path with at least 6 owned layers the exchange runs on
        its own stream and overlaps the interior work (`split_ranges`);
        otherwise exchange, then the whole local step."""
        if self._dev is not None and self.overlap_ok():
            self._overlapped_step()
            return
        halo_exchange(self.x, self.layout, self.group)
        self._local()

    # ---- halo exchange overlapped with the interior ------------------------
    def overlap_ok(self) -> bool:
        """The split step needs an interior (>= 6 owned layers), neighbours to
        wait for, and the overlap-safe update order (the default one-launch
        bulk reduce-add path; the deterministic colour order keeps the plain
        step)."""
        import os
        z0, z1 = self.layout.own
        return (self.layout.world > 1 and z1 - z0 >= 6
                and os.environ.get("DGB_SLAB_OVERLAP", "1") != "0"
                and "0" not in (os.environ.get("DGB_AVS_ATOMIC", "1"),
                                os.environ.get("DGB_AVS_ATOMIC_ORDER", "1")))

    def split_ranges(self) -> dict:
        """Layer ranges of the split step (global layer indices, half open).

        interior (needs owned x only, so it runs while the halo is in flight):
          residual on [z0+1, z1-1) (reads x on [z0, z1)); AVS patches with
          vertex v_z in [z0+3, z1-2) (read r on [v-1, v], write x on
          [z0+2, z1-3], layers no boundary residual reads) or ACS cells of
          [z0+2, z1-2);
        boundary (after the halo): residual on [z0-1, z0+1) and [z1-1, z1+1)
          (reads x on [z0-2, z0+2) and [z1-2, z1+2)), then the remaining
          patches v_z in [max(1,z0), z0+3) and [z1-2, min(nz-1,z1)+1), or
          cells [z0, z0+2) and [z1-2, z1).
        The union is exactly the plain step's work; the update order of a
        DoF changes only by the reduce-add order (rounding)."""
        z0, z1 = self.layout.own
        nz = self.layout.nz
        r_lo, r_hi = self.layout.res
        if self.kind == "avs":
            p_lo, p_hi = self.layout.pv[0], self.layout.pv[1] + 1
            inner = (z0 + 3, z1 - 2)
            outer = [(p_lo, inner[0]), (inner[1], p_hi)]
        else:
            inner = (z0 + 2, z1 - 2)
            outer = [(z0, inner[0]), (inner[1], z1)]
        return {"res_inner": (z0 + 1, z1 - 1),
                "res_outer": [(r_lo, z0 + 1), (z1 - 1, min(nz, r_hi))],
                "solve_inner": inner, "solve_outer": outer}

    def _split_part(self, part: str) -> None:
        from . import _lib
        from ._device import stream_handle

        dev = self._dev
        lib = dev._lib
        st = stream_handle()
        kind = _lib.KINDS[self.kind]
        rg = self.split_ranges()
        xp, bp, rp = self.x.data_ptr(), self.b.data_ptr(), self.r.data_ptr()
        if part == "interior":
            res, sol = [rg["res_inner"]], [rg["solve_inner"]]
        else:
            res, sol = rg["res_outer"], rg["solve_outer"]
        for lo, hi in res:
            if hi > lo:
                _lib.check(lib.dg_residual(dev.handle, xp, bp, rp, lo, hi, st))
        for lo, hi in sol:
            if hi > lo:
                _lib.check(lib.dg_solve_range(dev.handle, kind, self.omega, rp, xp, lo, hi, st))

    def _overlapped_step(self) -> None:
        cur = torch.cuda.current_stream()
        if not hasattr(self, "_comm"):
            self._comm = torch.cuda.Stream()
        comm = self._comm
        comm.wait_stream(cur)  # the previous step's updates of the sent layers
        plan = self.layout.halo_plan()
        with torch.cuda.stream(comm):
            ops = []
            for peer, send, recv in plan:
                ops.append(dist.P2POp(dist.isend, self.x[send], peer, self.group))
                ops.append(dist.P2POp(dist.irecv, self.x[recv], peer, self.group))
            works = dist.batch_isend_irecv(ops)
        self._split_part("interior")
        for w in works:
            w.wait()          # the current stream waits for the exchange
        cur.wait_stream(comm)
        self._split_part("boundary")

    def owned_x(self) -> torch.Tensor:
        return self.x[self.owned]

    # ---- bench instrumentation --------------------------------------------
    def launches_per_step(self) -> int:
        if self._dev is None:
            return 0
        return int(self._dev._lib.dg_last_launch_count(self._dev.handle))

    def kernel_times(self, reps: int = 5) -> dict:
        """Device time of the halo exchange, of the residual launch alone and
        of the local step as `dg_smooth` issues it (direct launches); solve =
        step - residual."""
        from . import _lib
        from ._device import stream_handle

        dev = self._dev
        lib = dev._lib
        st = stream_handle()
        lay = self.layout
        t_res = t_step = t_x = 0.0
        for rep in range(reps + 1):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record()
            halo_exchange(self.x, lay, self.group)
            ev[1].record()
            _lib.check(lib.dg_residual(dev.handle, self.x.data_ptr(), self.b.data_ptr(),
                                       self.r.data_ptr(), lay.res[0], lay.res[1], st))
            ev[2].record()
            _lib.check(lib.dg_smooth(dev.handle, _lib.KINDS[self.kind], self.omega, 0,
                                     self.x.data_ptr(), self.b.data_ptr(), self.r.data_ptr(),
                                     0, st))
            ev[3].record()
            torch.cuda.synchronize()
            if rep:
                t_x += ev[0].elapsed_time(ev[1])
                t_res += ev[1].elapsed_time(ev[2])
                t_step += ev[2].elapsed_time(ev[3])
        nl = int(lib.dg_last_launch_count(dev.handle))
        return {"halo_ms": t_x / reps, "residual_ms": t_res / reps,
                "solve_ms": (t_step - t_res) / reps, "step_direct_ms": t_step / reps,
                "residual_launches": 1, "solve_launches": nl - 1}

    def e2e(self, x_owned, b_owned, reps: int = 5) -> dict:
        """Public-API step with pinned host I/O of this rank's owned x, b."""
        xh = torch.from_numpy(np.ascontiguousarray(x_owned)).pin_memory()
        bh = torch.from_numpy(np.ascontiguousarray(b_owned)).pin_memory()
        own = self.owned
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        for it in range(reps + 1):
            if it == 1:
                dist.barrier(group=self.group)
                torch.cuda.synchronize()
                e0.record()
            self.x[own].copy_(xh, non_blocking=True)
            self.b[own].copy_(bh, non_blocking=True)
            halo_exchange(self.b, self.layout, self.group)
            self.step()
            xh.copy_(self.x[own], non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        n = self.n_owned
        return {"unit": "DoF/s", "ms_per_step": ms, "dofs_local": n,
                "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 8 * n,
                "api": "SlabSmoother.load/step with pinned host x, b (per rank)"}
