"""Matrix-free SIPG operator on uniform Cartesian levels (device).

Mirror of the reference's `dgmg.dgop` entry points on the hot path
(`pkg/src/dgmg/dgop.py`):

- `DofLayout` (`dgop.py:70-103`): cell-major canonical layout;
- `make_context` (`dgop.py:399-411`) -> `OperatorContext` (`254-275`);
- `apply_operator(ctx, u, out=None)` (`dgop.py:762-779`): v = A u,
  ValueError on a size mismatch;
- `residual(ctx, x, b, out)` (`dgop.py:782-788`): out = b - A x.

The arithmetic runs in `residual_kernel` (csrc/kernels.cuh) through the C ABI.
On a Cartesian level the reference's quadrature form equals the Kronecker
sum of 1D SIPG matrices, which is what the kernel applies.  Only Cartesian
levels are in scope (distorted meshes are SURVEY 8(f) "next").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._device import Staged, require_cuda, stream_handle
from .basis import Basis1D, sipg_penalty
from .flops import FlopCounter, operator_apply_flops
from .mesh import level_dims
from .tables import LevelTables, build_tables

__all__ = [
    "DofLayout",
    "OperatorContext",
    "penalty",
    "make_context",
    "apply_operator",
    "residual",
]


def penalty(gamma_hat: float, k: int, h_plus: float, h_minus: float) -> float:
    """`dgop.py:64-67`."""
    return sipg_penalty(gamma_hat, k, h_plus, h_minus)


@dataclass(frozen=True)
class DofLayout:
    """global index = cell*(k+1)^d + sum_t i_t (k+1)^(t-1) (`dgop.py:70-103`).
    `dims` generalises `ncells_dim` to boxes."""

    dim: int
    degree: int
    dims: tuple

    @property
    def ncells_dim(self) -> int:
        if len(set(self.dims)) != 1:
            raise ValueError("ncells_dim is defined for cube levels only")
        return self.dims[0]

    @property
    def n1d(self) -> int:
        return self.degree + 1

    @property
    def cell_dofs(self) -> int:
        return self.n1d ** self.dim

    @property
    def ncells(self) -> int:
        return int(np.prod(self.dims))

    @property
    def ndofs(self) -> int:
        return self.ncells * self.cell_dofs

    def node_shape(self) -> tuple:
        return (self.n1d,) * self.dim

    def grid_shape(self) -> tuple:
        return tuple(self.dims[::-1]) + self.node_shape()

    def global_index(self, cell: int, node_multi: tuple) -> int:
        i = sum(node_multi[t] * self.n1d ** t for t in range(self.dim))
        return cell * self.cell_dofs + i


def _as_basis(basis) -> Basis1D:
    if isinstance(basis, Basis1D):
        return basis
    k = int(basis.degree)
    quad = getattr(basis, "quad", None)
    nq = int(quad.n) if quad is not None else k + 1
    return Basis1D.make(k, nq)


def _level_h(level) -> float:
    if not getattr(level, "cartesian", True):
        raise NotImplementedError("device path supports Cartesian levels only")
    h = getattr(level, "h", None)
    if h is not None:
        return float(h)
    lengths = np.asarray(level.lengths, dtype=float)
    if not np.all(lengths == lengths[0]):
        raise NotImplementedError("device path needs equal cell lengths per direction")
    return float(lengths[0])


class OperatorContext:
    """Level + basis + device tables (`dgop.py:254-275`)."""

    def __init__(self, level, basis: Basis1D, layout: DofLayout, gamma_hat: float,
                 tables: LevelTables, counter: FlopCounter | None = None):
        self.level = level
        self.basis = basis
        self.layout = layout
        self.gamma_hat = gamma_hat
        self.tables = tables
        self.counter = counter
        self.ws = None
        self._dev = None

    @property
    def dev(self) -> _lib.DeviceLevel:
        """Device level (created lazily so host-only setup needs no GPU)."""
        if self._dev is None:
            require_cuda()
            self._dev = _lib.DeviceLevel(self.tables, self.layout.dims)
        return self._dev

    @property
    def ndofs(self) -> int:
        return self.layout.ndofs

    def new_vector(self) -> np.ndarray:
        return np.zeros(self.ndofs)

    def count(self, kernel: str, flops: float) -> None:
        if self.counter is not None:
            self.counter.add(kernel, flops)


def make_context(level, basis, gamma_hat: float = 1.0,
                 counter: FlopCounter | None = None, ws=None) -> OperatorContext:
    """`dgop.py:399-411`.  Accepts this package's or the reference's level and
    basis objects (duck-typed: dim, ncells_dim|dims, lengths|h; degree)."""
    b = _as_basis(basis)
    dims = level_dims(level)
    h = _level_h(level)
    layout = DofLayout(dim=len(dims), degree=b.degree, dims=tuple(dims))
    tables = build_tables(b, h, tuple(dims), gamma_hat,
                          with_patches=b.n <= 8 and min(dims) >= 2)
    return OperatorContext(level, b, layout, gamma_hat, tables, counter)


def _count_apply(ctx: OperatorContext, kernel: str) -> None:
    if ctx.counter is not None:
        lay = ctx.layout
        ctx.count(kernel, operator_apply_flops(lay.dim, lay.n1d, ctx.basis.qpts.size,
                                               lay.dims))


def apply_operator(ctx: OperatorContext, u, out=None,
                   kernel: str = "operator_apply"):
    """v = A u (`dgop.py:762-779`)."""
    dev = ctx.dev
    n = ctx.ndofs
    su = Staged(u, n, "u")
    if out is None:
        out = np.empty(n) if su.host is not None else su.dev.new_empty(n)
    sv = Staged(out, n, "out", need_copy=False)
    if sv.ptr == su.ptr:
        raise ValueError("apply_operator: out must not alias u")
    _lib.check(dev._lib.dg_apply(dev.handle, su.ptr, sv.ptr, 0, ctx.layout.dims[-1],
                                 stream_handle()))
    sv.finish()
    _count_apply(ctx, kernel)
    return out


def residual(ctx: OperatorContext, x, b, out, kernel: str = "residual"):
    """out = b - A x (`dgop.py:782-788`)."""
    dev = ctx.dev
    n = ctx.ndofs
    sx = Staged(x, n, "x")
    sb = Staged(b, n, "b")
    so = Staged(out, n, "out", need_copy=False)
    if so.ptr == sx.ptr:
        raise ValueError("residual: out must not alias x")
    _lib.check(dev._lib.dg_residual(dev.handle, sx.ptr, sb.ptr, so.ptr, 0,
                                    ctx.layout.dims[-1], stream_handle()))
    so.finish()
    _count_apply(ctx, kernel)
    ctx.count(kernel, ctx.ndofs)
    return out
