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
import torch

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
    "assemble_dense",
    "compute_rhs",
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
                          with_patches=min(dims) >= 2)
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


def _coupling(t: LevelTables) -> np.ndarray:
    """Rank-2 face coupling a_pm = alpha e_n e_1^T + beta e_n bg0^T +
    betap bg1 e_1^T (`polybasis.py:278-284`; GL end nodes are nodal)."""
    n = t.n
    a = np.zeros((n, n))
    a[n - 1, 0] += t.alpha
    a[n - 1, :] += t.beta * t.bg[0]
    a[:, 0] += t.betap * t.bg[1]
    return a


def global_1d_pencils(ctx: OperatorContext):
    """Per direction the global 1D matrices (A_g, M_g) of a Cartesian level:
    A_g block tridiagonal with A_diag(digit) on the diagonal and the rank-2
    coupling a_pm above it, M_g = I (x) M."""
    t = ctx.tables
    n, dims = ctx.layout.n1d, ctx.layout.dims
    apm = _coupling(t)
    out = []
    for dt in range(ctx.layout.dim):
        nt = dims[dt]
        a1 = np.zeros((nt * n, nt * n))
        for c in range(nt):
            digit = (1 if c == 0 else 0) | (2 if c == nt - 1 else 0)
            a1[c * n:(c + 1) * n, c * n:(c + 1) * n] = t.adiag[digit]
            if c + 1 < nt:
                a1[c * n:(c + 1) * n, (c + 1) * n:(c + 2) * n] = apm
                a1[(c + 1) * n:(c + 2) * n, c * n:(c + 1) * n] = apm.T
        out.append((a1, np.kron(np.eye(nt), t.mass)))
    return out


def assemble_dense(ctx: OperatorContext, via: str = "kronecker", device=None):
    """Dense level matrix in the canonical layout (cf. `dgop.py:1045-1072`),
    for coarse levels: on a Cartesian level A = sum_t M (x) .. A_g^(t) .. (x) M
    with block-tridiagonal 1D A_g, permuted from the
    direction-major to the canonical dof order.  Built with torch on `device`
    (the 1D factors are host setup); returns a numpy array when device is
    None.  `via="matvec"` assembles from device operator applications."""
    lay = ctx.layout
    ndofs = lay.ndofs
    if ndofs > 40000:
        raise ValueError("dense assembly limited to 40000 dofs")
    dev = torch.device(device) if device is not None else torch.device("cpu")
    if via == "matvec":
        eye = torch.eye(ndofs, dtype=torch.float64, device="cuda")
        a = torch.empty((ndofs, ndofs), dtype=torch.float64, device="cuda")
        for j in range(ndofs):
            apply_operator(ctx, eye[j], out=a[j])
        a = a.T.contiguous().to(dev)
        return a.numpy() if device is None else a
    if via not in ("kronecker", "quadrature"):
        raise ValueError("via must be 'kronecker', 'quadrature' or 'matvec'")
    d = lay.dim
    n, dims = lay.n1d, lay.dims
    ag, mg = [], []
    for a1, m1 in global_1d_pencils(ctx):
        ag.append(torch.from_numpy(a1).to(dev))
        mg.append(torch.from_numpy(m1).to(dev))
    a = None
    for dt in range(d):
        term = None
        for u in reversed(range(d)):          # kron order: slowest direction first
            f = ag[u] if u == dt else mg[u]
            term = f if term is None else torch.kron(term, f)
        a = term if a is None else a + term
    # canonical dof g = cell n^d + sum_t i_t n^(t-1) -> direction-major index
    shape = tuple(dims[::-1]) + (n,) * d
    idx = np.indices(shape).reshape(2 * d, -1)
    jdm = np.zeros(idx.shape[1], dtype=np.int64)
    stride = 1
    for dt in range(d):
        c_t = idx[d - 1 - dt]
        i_t = idx[2 * d - 1 - dt]
        jdm += (c_t * n + i_t) * stride
        stride *= dims[dt] * n
    perm = torch.from_numpy(jdm).to(dev)
    a = a.index_select(0, perm).index_select(1, perm)
    return a.numpy() if device is None else a


def mode_contract(t: torch.Tensor, mat: torch.Tensor, axis: int) -> torch.Tensor:
    """Contract `axis` of the contiguous fp64 CUDA tensor t with mat (I x K,
    K = t.shape[axis]): out[.., i, ..] = sum_k mat[i, k] t[.., k, ..], the
    axis staying in place (C ABI `dg_mode_contract`, csrc/coarse.cu)."""
    from ._device import stream_handle
    t = t.contiguous()
    mat = mat.contiguous()
    shape = list(t.shape)
    k = shape[axis]
    if mat.shape[1] != k:
        raise ValueError("mode_contract: matrix columns must match the contracted axis")
    outer = int(np.prod(shape[:axis], dtype=np.int64))
    inner = int(np.prod(shape[axis + 1:], dtype=np.int64))
    shape[axis] = mat.shape[0]
    out = torch.empty(shape, dtype=torch.float64, device=t.device)
    lib = _lib.load()
    _lib.check(lib.dg_mode_contract(t.data_ptr(), out.data_ptr(), mat.data_ptr(), outer, k,
                                    int(mat.shape[0]), inner, 0, stream_handle()))
    return out


def _contract_quad(w: torch.Tensor, vals: torch.Tensor, k: int) -> torch.Tensor:
    """(B, q_1..q_k) reversed quadrature layout -> (B, n_k..n_1) canonical:
    out[b, i_k..i_1] = sum_q prod_t phi_{i_t}(x_{q_t}) w[b, q_1..q_k]
    (`_tensor.backward_all`, `_tensor.py:81-97`): one hand-written mode
    contraction per direction, then the axis reversal to the canonical order."""
    y = w
    for ax in range(1, k + 1):
        y = mode_contract(y, vals, ax)      # (B, n_1, .., n_k) when done
    return y.permute(0, *range(k, 0, -1)).contiguous() if k > 1 else y


def compute_rhs(ctx: OperatorContext, f, g):
    """Load vector (`dgop.py:800-871`): volume source f plus the Nitsche
    boundary terms of the Dirichlet data g with the operator's penalty and
    trace weights, on a Cartesian level.  f and g are the reference's host
    callables on (N, d) coordinate arrays; their values at the quadrature
    points are contracted with the basis on the device (sum factorisation).
    Returns a numpy vector in the canonical layout."""
    require_cuda()
    lay = ctx.layout
    d, n, dims = lay.dim, lay.n1d, lay.dims
    b = ctx.basis
    h = float(ctx.tables.h)
    qp, qw = np.asarray(b.qpts, float), np.asarray(b.qwts, float)
    nq = qp.size
    dev = torch.device("cuda")
    vals = torch.from_numpy(np.ascontiguousarray(b.values)).to(dev)      # (n, nq)
    # cell origins, cell id order (direction 1 fastest)
    cidx = np.indices(tuple(dims[::-1])).reshape(d, -1)[::-1].T            # (ncells, d)
    origin = cidx * h
    # volume: reversed quadrature layout (q_1 slowest), column t = direction t+1
    ref = np.stack([g_.ravel() for g_ in np.meshgrid(*([qp] * d), indexing="ij")], axis=-1)
    wq = np.ones(1)
    for _ in range(d):
        wq = np.multiply.outer(wq, qw).ravel()
    coords = origin[:, None, :] + h * ref[None, :, :]
    fv = np.asarray(f(coords.reshape(-1, d)), dtype=float).reshape(lay.ncells, -1)
    w = torch.from_numpy(fv * (h ** d * wq)[None, :]).to(dev)
    rhs = _contract_quad(w.reshape((lay.ncells,) + (nq,) * d), vals, d)
    rhs = rhs.reshape(lay.ncells, -1)
    # boundary faces: Nitsche terms gamma_e |N| w g v + (-s) |N|/h w g dv/dn
    gamma_e = sipg_penalty(ctx.gamma_hat, lay.degree, h, h)
    area = h ** (d - 1)
    t_full = area / h
    bv = torch.from_numpy(np.asarray(b.bv, float)).to(dev)
    bg = torch.from_numpy(np.asarray(b.bg, float)).to(dev)
    for tau in range(1, d + 1):
        trans = [t for t in range(1, d + 1) if t != tau]
        if trans:
            tref = np.stack([g_.ravel() for g_ in np.meshgrid(*([qp] * len(trans)),
                                                               indexing="ij")], axis=-1)
            wf = np.ones(1)
            for _ in trans:
                wf = np.multiply.outer(wf, qw).ravel()
        else:
            tref, wf = np.zeros((1, 0)), np.ones(1)
        for p in (0, 1):
            sel = cidx[:, tau - 1] == (0 if p == 0 else dims[tau - 1] - 1)
            ids = np.nonzero(sel)[0]
            fref = np.empty((tref.shape[0], d))
            for j, t in enumerate(trans):
                fref[:, t - 1] = tref[:, j]
            fref[:, tau - 1] = float(p)
            fc = origin[ids][:, None, :] + h * fref[None, :, :]
            gv = np.asarray(g(fc.reshape(-1, d)), dtype=float).reshape(len(ids), -1)
            sign = 1.0 if p == 1 else -1.0
            mv = torch.from_numpy(gv * (gamma_e * area * wf)[None, :]).to(dev)
            mg = torch.from_numpy(gv * (-sign * t_full * wf)[None, :]).to(dev)
            k = len(trans)
            if k:
                tv = _contract_quad(mv.reshape((len(ids),) + (nq,) * k), vals, k)
                tg = _contract_quad(mg.reshape((len(ids),) + (nq,) * k), vals, k)
            else:
                tv, tg = mv, mg
            # contrib[c, nodes] with the normal node axis of tau inserted
            tv = tv.reshape((len(ids),) + (n,) * k)
            tg = tg.reshape((len(ids),) + (n,) * k)
            ax = 1 + (d - tau)  # canonical node axis of direction tau
            contrib = (tv.unsqueeze(ax) * bv[p].reshape([1] * ax + [n] + [1] * (d - ax))
                       + tg.unsqueeze(ax) * bg[p].reshape([1] * ax + [n] + [1] * (d - ax)))
            flat = rhs.view(lay.ncells, -1)
            flat[torch.from_numpy(ids).to(dev)] += contrib.reshape(len(ids), -1)
    return rhs.reshape(-1).cpu().numpy()
