"""Distorted (multilinear) meshes: the SIPG operator on non-Cartesian cells
(first part).

Mirror of the reference's non-Cartesian path:

- `distort(hierarchy, factor, rng_seed)` (`mesh.py:227-284`): every
  interior vertex of the coarse level moves by factor * h_v in a uniformly
  random direction (numpy PCG64 stream of the seed, as the reference draws
  it), finer levels by midpoint refinement (`mesh.py:160-182`);
- the multilinear geometry (`dgop.py:277-374`): per cell and volume
  quadrature point the symmetric metric detJ J^-1 J^-T w, per face and face
  quadrature point the penalty and the normal-derivative factors of both
  sides, per boundary face the Nitsche factors — host setup (numpy), uploaded
  once;
- `DistortedContext` + `apply_operator` / `residual`: v = A u by the
  sm_100a kernel `dist_apply_kernel<D, n>` (`csrc/dist_op.cu`): one CTA per
  cell, sum-factorised reference gradients at the quadrature points, the
  metric applied per point, the adjoint contractions; every face term is
  evaluated by both of its cells (each adds its own side), so there are no
  atomics (`dgop.py:432-481`, `583-759`, non-Cartesian branches).

The surrogate cell smoother on these meshes (`fastdiag.py:381-436`) is the
next step; it is not built yet.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._device import Staged, require_cuda, stream_handle
from .basis import Basis1D, sipg_penalty

__all__ = ["DistortedLevel", "DistortedHierarchy", "distort", "DistortedContext",
           "make_distorted_context", "apply_operator", "residual"]

_SYM = {2: [(0, 0), (1, 1), (0, 1)], 3: [(0, 0), (1, 1), (2, 2), (0, 1), (0, 2), (1, 2)]}


def cartesian_vertex_grid(d: int, n: int) -> np.ndarray:
    """(n+1,)*d + (d,) vertex coordinates; array axis a <-> direction d - a."""
    coords = np.linspace(0.0, 1.0, n + 1)
    grid = np.empty((n + 1,) * d + (d,))
    for t in range(1, d + 1):
        shape = [1] * d
        shape[d - t] = n + 1
        grid[..., t - 1] = coords.reshape(shape)
    return grid


def _refine(coarse: np.ndarray, d: int, n: int) -> np.ndarray:
    """Midpoint refinement: each fine vertex is the mean of the coarse
    vertices of the smallest coarse entity containing it."""
    fine = np.empty((2 * n + 1,) * d + (d,))
    for parity in range(2 ** d):
        s = [(parity >> t) & 1 for t in range(d)]
        target = tuple(slice(s[d - 1 - a], None, 2) for a in range(d))
        acc, cnt = None, 0
        for sub in range(2 ** d):
            o = [(sub >> t) & 1 for t in range(d)]
            if any(o[t] > s[t] for t in range(d)):
                continue
            src = tuple(slice(o[d - 1 - a], o[d - 1 - a] + n + 1 - s[d - 1 - a]) for a in range(d))
            acc = coarse[src].copy() if acc is None else acc + coarse[src]
            cnt += 1
        fine[target] = acc / cnt
    return fine


class DistortedLevel:
    """A multilinear cube level: n cells per direction, vertex grid."""

    cartesian = False

    def __init__(self, dim: int, n: int, vertex_grid: np.ndarray, index: int = 0):
        self.dim, self.ncells_dim, self.index = dim, n, index
        self.dims = (n,) * dim
        self.vertex_grid = vertex_grid
        self.ncells = n ** dim

    def cell_corners(self) -> np.ndarray:
        """(ncells, 2^d, d), corner c = sum_t s_t 2^t, cell ids v_1 fastest."""
        d, n = self.dim, self.ncells_dim
        out = np.empty((2 ** d,) + (n,) * d + (d,))
        for c in range(2 ** d):
            s = [(c >> t) & 1 for t in range(d)]
            out[c] = self.vertex_grid[tuple(slice(s[d - 1 - a], s[d - 1 - a] + n)
                                            for a in range(d))]
        return np.ascontiguousarray(np.moveaxis(out, 0, -2).reshape(self.ncells, 2 ** d, d))


class DistortedHierarchy:
    def __init__(self, dim, levels):
        self.dim, self.levels = dim, levels


def distort(hierarchy, factor: float, rng_seed: int) -> DistortedHierarchy:
    """`mesh.py:227-284` for cube hierarchies (this package's or the reference's)."""
    if not 0.0 <= factor < 0.5:
        raise ValueError("distortion factor must be in [0, 0.5)")
    d = hierarchy.levels[0].dim
    n = hierarchy.levels[0].ncells_dim if hasattr(hierarchy.levels[0], "ncells_dim") \
        else hierarchy.levels[0].dims[0]
    base = cartesian_vertex_grid(d, n)
    grid = base.copy()
    h_v = np.full((n + 1,) * d, np.inf)
    for ax in range(d):
        edge = np.linalg.norm(np.diff(base, axis=ax), axis=-1)
        lo = [slice(None)] * d
        hi = [slice(None)] * d
        lo[ax], hi[ax] = slice(0, n), slice(1, n + 1)
        np.minimum.at(h_v, tuple(lo), edge)
        np.minimum.at(h_v, tuple(hi), edge)
    interior = np.ones((n + 1,) * d, dtype=bool)
    for ax in range(d):
        sl = [slice(None)] * d
        sl[ax] = [0, n]
        interior[tuple(sl)] = False
    rng = np.random.default_rng(rng_seed)
    n_int = int(interior.sum())
    dirs = rng.standard_normal((n_int, d))
    norms = np.linalg.norm(dirs, axis=1, keepdims=True)
    while np.any(norms < 1e-12):
        redraw = norms[:, 0] < 1e-12
        dirs[redraw] = rng.standard_normal((int(redraw.sum()), d))
        norms = np.linalg.norm(dirs, axis=1, keepdims=True)
    dirs /= norms
    grid[interior] += factor * h_v[interior, None] * dirs
    levels = [DistortedLevel(d, n, grid, 0)]
    for lv in range(1, len(hierarchy.levels)):
        prev = levels[-1]
        levels.append(DistortedLevel(d, 2 * prev.ncells_dim,
                                     _refine(prev.vertex_grid, d, prev.ncells_dim), lv))
    return DistortedHierarchy(d, levels)


# ------------------------------------------------------------------ geometry
def _grad_table(d: int, ref: np.ndarray) -> np.ndarray:
    """(2^d, Q, d) gradients of the multilinear corner shape functions."""
    q = ref.shape[0]
    out = np.empty((2 ** d, q, d))
    for c in range(2 ** d):
        s = [(c >> t) & 1 for t in range(d)]
        for t in range(d):
            g = np.ones(q)
            for u in range(d):
                x = ref[:, u]
                g = g * ((1.0 if s[u] else -1.0) if u == t else (x if s[u] else 1.0 - x))
            out[c, :, t] = g
    return out


def _adjugate(j: np.ndarray) -> np.ndarray:
    d = j.shape[-1]
    adj = np.empty_like(j)
    if d == 2:
        adj[..., 0, 0], adj[..., 1, 1] = j[..., 1, 1], j[..., 0, 0]
        adj[..., 0, 1], adj[..., 1, 0] = -j[..., 0, 1], -j[..., 1, 0]
        return adj
    for r in range(3):
        for c in range(3):
            r1, r2 = [x for x in range(3) if x != c]
            c1, c2 = [x for x in range(3) if x != r]
            v = j[..., r1, c1] * j[..., r2, c2] - j[..., r1, c2] * j[..., r2, c1]
            adj[..., r, c] = -v if (r + c) % 2 else v
    return adj


def _det(j: np.ndarray) -> np.ndarray:
    if j.shape[-1] == 2:
        return j[..., 0, 0] * j[..., 1, 1] - j[..., 0, 1] * j[..., 1, 0]
    return np.linalg.det(j)


def _tensor_points(pts: np.ndarray, k: int) -> np.ndarray:
    """(nq^k, k) points, first coordinate slowest (the reversed layout)."""
    if k == 0:
        return np.zeros((1, 0))
    g = np.meshgrid(*([pts] * k), indexing="ij")
    return np.stack([a.ravel() for a in g], axis=-1)


def _tensor_weights(w: np.ndarray, k: int) -> np.ndarray:
    out = np.ones(1)
    for _ in range(k):
        out = np.multiply.outer(out, w).ravel()
    return out


class DistortedGeometry:
    """Host geometry of a multilinear level, packed for the device kernel.

    metric:   (B, Q, S)       detJ J^-1 J^-T w (symmetric pairs `_SYM`)
    faces[t]: (F_t, qf, 1+2d) [pen_half, t_plus(d), t_minus(d)] interior
    bnd[t][p]:(F_b, qf, 1+d)  [pen_bnd, t_bnd(d)] boundary side p
    """

    def __init__(self, level: DistortedLevel, basis: Basis1D, gamma_hat: float):
        d, n, k = level.dim, level.ncells_dim, basis.degree
        pts, w = np.asarray(basis.qpts, float), np.asarray(basis.qwts, float)
        corners = level.cell_corners()
        ref = _tensor_points(pts, d)
        wq = _tensor_weights(w, d)
        dn = _grad_table(d, ref)
        jac = np.einsum("fcx,cqt->fqxt", corners, dn)
        det = _det(jac)
        if np.any(det <= 0.0):
            raise ValueError("nonpositive Jacobian at a quadrature point")
        adj = _adjugate(jac)
        g = np.einsum("fqxt,fqxs->fqts", adj, adj)
        self.metric = np.empty(det.shape + (len(_SYM[d]),))
        for j_, (a, b) in enumerate(_SYM[d]):
            self.metric[:, :, j_] = g[:, :, a, b] / det * wq
        cellvol = (det * wq).sum(axis=1)
        cgrid = corners.reshape((n,) * d + (2 ** d, d))
        vgrid = cellvol.reshape((n,) * d)
        wf = _tensor_weights(w, d - 1)
        self.faces, self.bnd = [], []
        for tau in range(1, d + 1):
            ax = d - tau
            trans = [t for t in range(1, d + 1) if t != tau]

            def fref(side):
                tp = _tensor_points(pts, d - 1)
                out = np.empty((tp.shape[0], d))
                for j_, t in enumerate(trans):
                    out[:, t - 1] = tp[:, j_]
                out[:, tau - 1] = side
                return out

            def slab(arr, sl_ax):
                s = [slice(None)] * d
                s[ax] = sl_ax
                return arr[tuple(s)]

            dn_l, dn_r = _grad_table(d, fref(1.0)), _grad_table(d, fref(0.0))
            cl = slab(cgrid, slice(0, n - 1)).reshape(-1, 2 ** d, d)
            cr = slab(cgrid, slice(1, n)).reshape(-1, 2 ** d, d)
            vl = slab(vgrid, slice(0, n - 1)).ravel()
            vr = slab(vgrid, slice(1, n)).ravel()
            jl = np.einsum("fcx,cqt->fqxt", cl, dn_l)
            jr = np.einsum("fcx,cqt->fqxt", cr, dn_r)
            adl, adr = _adjugate(jl), _adjugate(jr)
            nvec = adl[:, :, tau - 1, :]
            nn = np.linalg.norm(nvec, axis=-1)
            area = (nn * wf).sum(axis=1)
            ge = gamma_hat * k * (k + 1) * (area / vl + area / vr)
            pack = np.empty(nn.shape + (1 + 2 * d,))
            pack[..., 0] = 0.5 * ge[:, None] * nn * wf
            pack[..., 1:1 + d] = np.einsum("fqts,fqs->fqt", adl, nvec) / _det(jl)[..., None] \
                * (0.5 * wf)[None, :, None]
            pack[..., 1 + d:] = np.einsum("fqts,fqs->fqt", adr, nvec) / _det(jr)[..., None] \
                * (0.5 * wf)[None, :, None]
            self.faces.append(pack)
            sides = []
            for p, (sl_ax, dnb, sign) in enumerate(((slice(0, 1), dn_r, -1.0),
                                                    (slice(n - 1, n), dn_l, 1.0))):
                cb = slab(cgrid, sl_ax).reshape(-1, 2 ** d, d)
                jb = np.einsum("fcx,cqt->fqxt", cb, dnb)
                adb = _adjugate(jb)
                nb = sign * adb[:, :, tau - 1, :]
                nbn = np.linalg.norm(nb, axis=-1)
                area_b = (nbn * wf).sum(axis=1)
                ge_b = gamma_hat * k * (k + 1) * (2.0 * area_b / slab(vgrid, sl_ax).ravel())
                pb = np.empty(nbn.shape + (1 + d,))
                pb[..., 0] = ge_b[:, None] * nbn * wf
                pb[..., 1:] = np.einsum("fqts,fqs->fqt", adb, nb) / _det(jb)[..., None] \
                    * wf[None, :, None]
                sides.append(pb)
            self.bnd.append(sides)


class DistortedContext:
    """Level + basis + device geometry for the multilinear operator."""

    def __init__(self, level: DistortedLevel, basis: Basis1D, gamma_hat: float = 4.0):
        if level.dim not in (2, 3):
            raise NotImplementedError("distorted device operator: dim 2 or 3")
        if basis.qpts.size != basis.n:
            raise NotImplementedError("distorted device operator: n_q = k + 1 quadrature")
        self.level, self.basis, self.gamma_hat = level, basis, gamma_hat
        self.dim, self.n = level.dim, basis.n
        self.ndofs = level.ncells * basis.n ** level.dim
        self.geom = DistortedGeometry(level, basis, gamma_hat)
        self._dev = None

    def _device(self):
        if self._dev is None:
            require_cuda()
            dev = torch.device("cuda")
            g = self.geom
            t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)  # noqa: E731
            self._dev = {
                "metric": t(g.metric),
                "faces": [t(f) for f in g.faces],
                "bnd": [[t(s) for s in sides] for sides in g.bnd],
                "vals": np.ascontiguousarray(self.basis.values.T),   # (nq, n): V[q][i]
                "grads": np.ascontiguousarray(self.basis.grads.T),   # (nq, n): D[q][i]
                "bv": np.ascontiguousarray(self.basis.bv),
                "bg": np.ascontiguousarray(self.basis.bg),
            }
        return self._dev


def make_distorted_context(level, basis, gamma_hat: float = 4.0) -> DistortedContext:
    b = basis if isinstance(basis, Basis1D) else Basis1D.make(int(basis.degree))
    return DistortedContext(level, b, gamma_hat)


class _DistArgs(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("degree", ctypes.c_int), ("ncells_dim", ctypes.c_int),
                ("metric", ctypes.c_void_p), ("faces", ctypes.c_void_p * 3),
                ("bnd", ctypes.c_void_p * 6), ("vals", ctypes.POINTER(ctypes.c_double)),
                ("grads", ctypes.POINTER(ctypes.c_double)), ("bv", ctypes.POINTER(ctypes.c_double)),
                ("bg", ctypes.POINTER(ctypes.c_double))]


def _args(ctx: DistortedContext) -> _DistArgs:
    dv = ctx._device()
    a = _DistArgs()
    a.dim, a.degree, a.ncells_dim = ctx.dim, ctx.basis.degree, ctx.level.ncells_dim
    a.metric = dv["metric"].data_ptr()
    for t in range(ctx.dim):
        a.faces[t] = dv["faces"][t].data_ptr()
        for p in range(2):
            a.bnd[2 * t + p] = dv["bnd"][t][p].data_ptr()
    dp = ctypes.POINTER(ctypes.c_double)
    a.vals = dv["vals"].ctypes.data_as(dp)
    a.grads = dv["grads"].ctypes.data_as(dp)
    a.bv = dv["bv"].ctypes.data_as(dp)
    a.bg = dv["bg"].ctypes.data_as(dp)
    return a


def apply_operator(ctx: DistortedContext, u, out=None):
    """v = A u on a multilinear level (`dgop.py:762-779`, non-Cartesian)."""
    lib = _lib.load()
    n = ctx.ndofs
    su = Staged(u, n, "u")
    if out is None:
        out = np.empty(n) if su.host is not None else su.dev.new_empty(n)
    sv = Staged(out, n, "out", need_copy=False)
    if sv.ptr == su.ptr:
        raise ValueError("apply_operator: out must not alias u")
    a = _args(ctx)
    _lib.check(lib.dg_dist_apply(ctypes.byref(a), su.ptr, None, sv.ptr, stream_handle()))
    sv.finish()
    return out


def residual(ctx: DistortedContext, x, b, out):
    """out = b - A x on a multilinear level (`dgop.py:782-788`)."""
    lib = _lib.load()
    n = ctx.ndofs
    sx, sb = Staged(x, n, "x"), Staged(b, n, "b")
    so = Staged(out, n, "out", need_copy=False)
    if so.ptr == sx.ptr:
        raise ValueError("residual: out must not alias x")
    a = _args(ctx)
    _lib.check(lib.dg_dist_apply(ctypes.byref(a), sx.ptr, sb.ptr, so.ptr, stream_handle()))
    so.finish()
    return out
