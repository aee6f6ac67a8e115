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
  atomics (`dgop.py:432-481`, `583-759`, non-Cartesian branches);
- `SurrogateCellSolverSet` (`fastdiag.py:381-436`, `457-496`): per cell and
  direction the 1D SIPG pencil of the cell's surrogate box (edge-averaged
  lengths, `mesh.py:436-458`), eigenpairs batched on the host (the north
  star keeps the 1D eigenproblems there), the per-cell fast-diagonalisation
  solves on the device (`dist_cell_fdm_kernel`);
- `DistortedSmoother` (ACS / MCS, `smoothers.py:131-166`; vertex patches
  need Cartesian geometry in the reference too), `compute_rhs`
  (`dgop.py:800-871`, multilinear branch) and the hooks the V-cycle uses.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._device import Staged, require_cuda, stream_handle
from .basis import Basis1D, sipg_penalty

__all__ = ["DistortedLevel", "DistortedHierarchy", "distort", "DistortedContext",
           "make_distorted_context", "apply_operator", "residual", "surrogate_lengths",
           "SurrogateCellSolverSet", "DistortedSmoother", "compute_rhs", "assemble_dense"]

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


def _adjugate(j):
    """Adjugate of (..., d, d) (numpy or torch), adj = det J^-1."""
    d = j.shape[-1]
    adj = j.new_empty(j.shape) if isinstance(j, torch.Tensor) else np.empty_like(j)
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


def _det(j):
    if j.shape[-1] == 2:
        return j[..., 0, 0] * j[..., 1, 1] - j[..., 0, 1] * j[..., 1, 0]
    return torch.linalg.det(j) if isinstance(j, torch.Tensor) else np.linalg.det(j)


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
    """Geometry of a multilinear level, packed for the device kernel and
    computed with torch on `device` (the GPU by default: a 16.8M-dof level's
    geometry costs seconds in numpy).

    metric:   (B, Q, S)       detJ J^-1 J^-T w (symmetric pairs `_SYM`)
    detjw:    (B, Q)          detJ w (load vector)
    faces[t]: (F_t, qf, 1+2d) [pen_half, t_plus(d), t_minus(d)] interior
    bnd[t][p]:(F_b, qf, 1+d)  [pen_bnd, t_bnd(d)] boundary side p
    """

    def __init__(self, level: DistortedLevel, basis: Basis1D, gamma_hat: float, device=None):
        if device is None:
            device = "cuda" if torch.cuda.is_available() else "cpu"
        dev = torch.device(device)
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)  # noqa: E731
        d, n, k = level.dim, level.ncells_dim, basis.degree
        pts, w = np.asarray(basis.qpts, float), np.asarray(basis.qwts, float)
        corners = T(level.cell_corners())
        ref = _tensor_points(pts, d)
        wq = T(_tensor_weights(w, d))
        jac = torch.einsum("fcx,cqt->fqxt", corners, T(_grad_table(d, ref)))
        det = _det(jac)
        if bool(torch.any(det <= 0.0)):
            raise ValueError("nonpositive Jacobian at a quadrature point")
        adj = _adjugate(jac)
        self.detjw = det * wq
        self.ref = ref
        g = torch.einsum("fqxt,fqxs->fqts", adj, adj)
        self.metric = torch.stack([g[:, :, a, b] / det * wq for a, b in _SYM[d]], dim=-1)
        del jac, adj, g
        cellvol = self.detjw.sum(dim=1)
        cgrid = corners.reshape((n,) * d + (2 ** d, d))
        vgrid = cellvol.reshape((n,) * d)
        wf = T(_tensor_weights(w, d - 1))
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
                s_ = [slice(None)] * d
                s_[ax] = sl_ax
                return arr[tuple(s_)]

            dn_l, dn_r = T(_grad_table(d, fref(1.0))), T(_grad_table(d, fref(0.0)))
            cl = slab(cgrid, slice(0, n - 1)).reshape(-1, 2 ** d, d)
            cr = slab(cgrid, slice(1, n)).reshape(-1, 2 ** d, d)
            vl = slab(vgrid, slice(0, n - 1)).reshape(-1)
            vr = slab(vgrid, slice(1, n)).reshape(-1)
            jl = torch.einsum("fcx,cqt->fqxt", cl, dn_l)
            jr = torch.einsum("fcx,cqt->fqxt", cr, dn_r)
            adl, adr = _adjugate(jl), _adjugate(jr)
            nvec = adl[:, :, tau - 1, :]
            nn = torch.linalg.vector_norm(nvec, dim=-1)
            area = (nn * wf).sum(dim=1)
            ge = gamma_hat * k * (k + 1) * (area / vl + area / vr)
            pack = torch.empty(nn.shape + (1 + 2 * d,), dtype=torch.float64, device=dev)
            pack[..., 0] = 0.5 * ge[:, None] * nn * wf
            pack[..., 1:1 + d] = torch.einsum("fqts,fqs->fqt", adl, nvec) / _det(jl)[..., None] \
                * (0.5 * wf)[None, :, None]
            pack[..., 1 + d:] = torch.einsum("fqts,fqs->fqt", adr, nvec) / _det(jr)[..., None] \
                * (0.5 * wf)[None, :, None]
            self.faces.append(pack)
            sides = []
            for p, (sl_ax, dnb, sign) in enumerate(((slice(0, 1), dn_r, -1.0),
                                                    (slice(n - 1, n), dn_l, 1.0))):
                cb = slab(cgrid, sl_ax).reshape(-1, 2 ** d, d)
                jb = torch.einsum("fcx,cqt->fqxt", cb, dnb)
                adb = _adjugate(jb)
                nb = sign * adb[:, :, tau - 1, :]
                nbn = torch.linalg.vector_norm(nb, dim=-1)
                area_b = (nbn * wf).sum(dim=1)
                ge_b = gamma_hat * k * (k + 1) * (2.0 * area_b / slab(vgrid, sl_ax).reshape(-1))
                pb = torch.empty(nbn.shape + (1 + d,), dtype=torch.float64, device=dev)
                pb[..., 0] = ge_b[:, None] * nbn * wf
                pb[..., 1:] = torch.einsum("fqts,fqs->fqt", adb, nb) / _det(jb)[..., None] \
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
        from .dgop import DofLayout
        self.level, self.basis, self.gamma_hat = level, basis, gamma_hat
        self.dim, self.n = level.dim, basis.n
        self.ndofs = level.ncells * basis.n ** level.dim
        self.layout = DofLayout(dim=level.dim, degree=basis.degree, dims=tuple(level.dims))
        self.counter = None
        self.geom = DistortedGeometry(level, basis, gamma_hat)
        self._dev = None

    def _device(self):
        if self._dev is None:
            require_cuda()
            dev = torch.device("cuda")
            g = self.geom
            t = lambda a: a.to(dev).contiguous()  # noqa: E731
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


def assemble_dense(ctx: DistortedContext, device="cuda") -> torch.Tensor:
    """Dense level matrix from device operator applications (coarse levels)."""
    n = ctx.ndofs
    if n > 40000:
        raise ValueError("dense assembly limited to 40000 dofs")
    eye = torch.eye(n, dtype=torch.float64, device="cuda")
    a = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for j in range(n):
        apply_operator(ctx, eye[j], out=a[j])
    return a.T.contiguous().to(device)


# ------------------------------------------------------------ cell smoother
def surrogate_lengths(corners: np.ndarray) -> np.ndarray:
    """Per direction the mean length of the 2^(d-1) edges aligned with it."""
    d = corners.shape[-1]
    out = np.empty(corners.shape[:-2] + (d,))
    for t in range(d):
        ls = [np.linalg.norm(corners[..., c + (1 << t), :] - corners[..., c, :], axis=-1)
              for c in range(2 ** d) if not (c >> t) & 1]
        st = np.stack(ls, axis=-1)
        if np.any(st <= 0.0):
            raise ValueError("degenerate (zero-length) edge")
        out[..., t] = st.mean(axis=-1)
    return out


def _eigh_batched(c):
    """Batched symmetric eigensolve of small matrices: cuSOLVER in chunks, the
    host LAPACK for any chunk cuSOLVER's batched path rejects (it fails on
    large batches of tiny matrices on this stack)."""
    lams, vs = [], []
    step = 4096
    for i in range(0, c.shape[0], step):
        blk = c[i:i + step].contiguous()
        try:
            lam, v = torch.linalg.eigh(blk)
        except RuntimeError:
            ln, vn = np.linalg.eigh(blk.cpu().numpy())
            lam, v = torch.from_numpy(ln).to(c.device), torch.from_numpy(vn).to(c.device)
        lams.append(lam)
        vs.append(v)
    return torch.cat(lams), torch.cat(vs)


def _batched_geneig(a, m):
    """Z^T A Z = diag(lam), Z^T M Z = I for stacks (B, n, n): Cholesky
    reduction + symmetric eigensolve (torch: batched on the device)."""
    chol = torch.linalg.cholesky(m)
    c = torch.linalg.solve_triangular(chol, a, upper=False)
    c = torch.linalg.solve_triangular(chol, c.transpose(1, 2), upper=False)
    c = 0.5 * (c + c.transpose(1, 2))
    lam, v = _eigh_batched(c)
    return torch.linalg.solve_triangular(chol.transpose(1, 2), v, upper=True), lam


class SurrogateCellSolverSet:
    """Per-cell surrogate fast-diagonalisation solvers (`fastdiag.py:381-436`)."""

    kind = "cell"

    def __init__(self, ctx: DistortedContext):
        from .fastdiag import SingularLocalSolverError
        lvl, b = ctx.level, ctx.basis
        d, n, nn, k = lvl.dim, lvl.ncells_dim, b.n, b.degree
        self.ctx, self.dim, self.n1 = ctx, d, nn
        dev = torch.device("cuda")
        hbar = torch.as_tensor(surrogate_lengths(lvl.cell_corners()), device=dev)
        B = lvl.ncells
        w = np.asarray(b.qwts, float)
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)  # noqa: E731
        mref = T((b.values * w) @ b.values.T)
        lref = T((b.grads * w) @ b.grads.T)
        bv, bg = b.bv, b.bg
        zs, lams = [], []
        ids = torch.arange(B, device=dev)
        for t in range(d):
            pos = (ids // n ** t) % n
            h = hbar[:, t]
            ge = ctx.gamma_hat * k * (k + 1) * (2.0 / h)
            one, half = torch.ones_like(h), torch.full_like(h, 0.5)
            eta = (torch.where(pos == 0, one, half), torch.where(pos == n - 1, one, half))
            a = lref[None] / h[:, None, None]
            for p in (0, 1):
                g1 = T((-1.0 if p == 0 else 1.0) * np.outer(bv[p], bg[p]))
                a = a + (ge * eta[p])[:, None, None] * T(np.outer(bv[p], bv[p]))[None] \
                    - (eta[p] / h)[:, None, None] * (g1 + g1.T)[None]
            z, lam = _batched_geneig(a, h[:, None, None] * mref[None])
            zs.append(z)
            lams.append(lam)
        inv = None
        for t in range(d):
            shape = [B] + [1] * d
            shape[1 + t] = nn
            arr = lams[t].reshape(shape)
            inv = arr if inv is None else inv + arr
        if bool(torch.any(inv <= 0.0)):
            raise SingularLocalSolverError("nonpositive Kronecker-sum eigenvalue")
        self._z = torch.stack(zs).contiguous()
        self._inv = (1.0 / inv).reshape(B, -1).contiguous()
        self.ncells = B

    def solve_partitioned(self, x, r, parts, omega: float) -> None:
        """x[cells] += omega A_c^-1 r_c for the given cell ids (None = all)."""
        lib = _lib.load()
        n = self.ctx.ndofs
        sx, sr = Staged(x, n, "x"), Staged(r, n, "r")
        ids = None
        cnt = 0
        if parts is not None:
            ids = torch.as_tensor(np.asarray(parts, dtype=np.int32)).cuda()
            cnt = int(ids.numel())
            if cnt == 0:
                sx.finish()
                return
        _lib.check(lib.dg_dist_cell_fdm(self.dim, self.n1 - 1, self.ncells, self._z.data_ptr(),
                                        self._inv.data_ptr(), sr.ptr, sx.ptr, float(omega),
                                        None if ids is None else ids.data_ptr(), cnt,
                                        stream_handle()))
        sx.finish()


class DistortedSmoother:
    """ACS / MCS smoothing steps on a multilinear level (`smoothers.py:131-166`)."""

    def __init__(self, ctx: DistortedContext, config):
        if config.kind not in ("acs", "mcs"):
            raise ValueError("vertex-patch smoothers require Cartesian geometry")
        self.ctx, self.config = ctx, config
        self.set = SurrogateCellSolverSet(ctx)
        n = ctx.level.ncells_dim
        ids = np.arange(ctx.level.ncells)
        par = np.zeros(ctx.level.ncells, dtype=np.int64)
        rem = ids.copy()
        for _ in range(ctx.dim):
            par += rem % n
            rem //= n
        self.colors = [ids] if config.kind == "acs" else \
            [s for s in (ids[par % 2 == 0], ids[par % 2 == 1]) if len(s)]
        self._parts = [None] if config.kind == "acs" else \
            [torch.as_tensor(c.astype(np.int32)).cuda() for c in self.colors]
        self.all_parts = None
        self._r = torch.empty(ctx.ndofs, dtype=torch.float64, device="cuda")
        self.use_graph = False

    def _solve(self, x, part, omega):
        lib = _lib.load()
        s = self.set
        cnt = 0 if part is None else int(part.numel())
        _lib.check(lib.dg_dist_cell_fdm(s.dim, s.n1 - 1, s.ncells, s._z.data_ptr(),
                                        s._inv.data_ptr(), self._r.data_ptr(), x.data_ptr(),
                                        float(omega), None if part is None else part.data_ptr(),
                                        cnt, stream_handle()))

    def smooth(self, x, b, reverse: bool = False) -> None:
        n = self.ctx.ndofs
        sx, sb = Staged(x, n, "x"), Staged(b, n, "b")
        om = self.config.omega
        if self.config.kind == "acs":
            residual(self.ctx, sx.dev, sb.dev, self._r)
            self._solve(sx.dev, None, om)
        else:
            order = range(len(self._parts))
            for c in (reversed(order) if reverse else order):
                residual(self.ctx, sx.dev, sb.dev, self._r)
                self._solve(sx.dev, self._parts[c], om)
        sx.finish()


# ---------------------------------------------------------------- load vector
def _corner_values(d: int, ref: np.ndarray) -> np.ndarray:
    out = np.ones((2 ** d, ref.shape[0]))
    for c in range(2 ** d):
        for t in range(d):
            x = ref[:, t]
            out[c] = out[c] * (x if (c >> t) & 1 else 1.0 - x)
    return out


def compute_rhs(ctx: DistortedContext, f, g) -> np.ndarray:
    """Load vector on a multilinear level (`dgop.py:800-871`): source f at the
    mapped Gauss points times detJ w, Nitsche boundary terms of g with the
    boundary penalty and the full normal-derivative factors; the basis
    contractions run on the device."""
    from .dgop import _contract_quad
    lvl, b, geo = ctx.level, ctx.basis, ctx.geom
    d, n, nn = lvl.dim, lvl.ncells_dim, b.n
    pts = np.asarray(b.qpts, float)
    dev = torch.device("cuda")
    vals = torch.from_numpy(np.ascontiguousarray(b.values)).to(dev)   # (n, nq)
    grads = torch.from_numpy(np.ascontiguousarray(b.grads)).to(dev)
    corners = lvl.cell_corners()
    coords = np.einsum("fcx,cq->fqx", corners, _corner_values(d, geo.ref))
    fv = np.asarray(f(coords.reshape(-1, d)), dtype=float).reshape(lvl.ncells, -1) \
        * geo.detjw.cpu().numpy()
    w = torch.from_numpy(fv).to(dev).reshape((lvl.ncells,) + (nn,) * d)
    rhs = _contract_quad(w, vals, d).reshape(lvl.ncells, -1)
    cidx = np.indices((n,) * d).reshape(d, -1)[::-1].T                  # (ncells, d), v_1 first
    bv = torch.from_numpy(np.asarray(b.bv, float)).to(dev)
    bg = torch.from_numpy(np.asarray(b.bg, float)).to(dev)
    for tau in range(1, d + 1):
        trans = [t for t in range(1, d + 1) if t != tau]
        tp = _tensor_points(pts, d - 1)
        for p in (0, 1):
            ids = np.nonzero(cidx[:, tau - 1] == (0 if p == 0 else n - 1))[0]
            fref = np.empty((tp.shape[0], d))
            for j_, t in enumerate(trans):
                fref[:, t - 1] = tp[:, j_]
            fref[:, tau - 1] = float(p)
            fc = np.einsum("fcx,cq->fqx", corners[ids], _corner_values(d, fref))
            gv = np.asarray(g(fc.reshape(-1, d)), dtype=float).reshape(len(ids), -1)
            pack = geo.bnd[tau - 1][p].cpu().numpy()                       # (Fb, qf, 1 + d)
            mv = torch.from_numpy(gv * pack[..., 0]).to(dev)
            mom = [torch.from_numpy(-gv * pack[..., 1 + t]).to(dev) for t in range(d)]
            k_ = len(trans)
            nf = len(ids)
            if k_ == 0:
                tv, tg = mv.reshape(nf), mom[tau - 1].reshape(nf)
            else:
                shp = (nf,) + (nn,) * k_
                tv = _contract_quad(mv.reshape(shp), vals, k_)
                for j_, t in enumerate(trans):
                    # tangential moment: derivative table along t, values elsewhere
                    y = mom[t - 1].reshape(shp)
                    for a_ in range(k_):
                        y = torch.tensordot(y, grads if a_ == j_ else vals, dims=([1], [1]))
                    tv = tv + (y.permute(0, *range(k_, 0, -1)) if k_ > 1 else y)
                tg = _contract_quad(mom[tau - 1].reshape(shp), vals, k_)
            tv = tv.reshape((nf,) + (nn,) * k_)
            tg = tg.reshape((nf,) + (nn,) * k_)
            ax = 1 + (d - tau)
            shape = [1] * ax + [nn] + [1] * (d - ax)
            contrib = tv.unsqueeze(ax) * bv[p].reshape(shape) + tg.unsqueeze(ax) * bg[p].reshape(shape)
            rhs[torch.from_numpy(ids).to(dev)] += contrib.reshape(nf, -1)
    return rhs.reshape(-1).cpu().numpy()
