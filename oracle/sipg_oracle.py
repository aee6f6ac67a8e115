"""CPU oracle for the fp64 Schwarz smoothing step -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` / `--impl reference`
legs may import it.  The package `paper_1910_11239_b200` never does.

It restates the reference's algorithm (`/root/reference/pkg/src/dgmg`) in
plain numpy, in the Kronecker-sum form of SURVEY App. A.5 (a different
contraction order than the reference's quadrature chains), on boxes as well
as cubes:

- 1D basis / factors / eigenpairs: `polybasis.py:48-341`;
- operator A = sum_t M x .. x A_g^(t) x .. x M with block-tridiagonal A_g
  (cell stiffness blocks `polybasis.py:247-259`, coupling a_pm
  `polybasis.py:278-284`), equal to `dgop.apply_operator` (`dgop.py:762-779`);
- residual `dgop.py:782-788`;
- cell / patch fast-diagonalisation solves `fastdiag.py:89-133`, `457-496`,
  `602-628`, index maps `fastdiag.py:546-582`, `mesh.py:297-326`;
- colourings `mesh.py:350-375`; smoothing steps `smoothers.py:131-166`;
- multigrid: 1D embeddings `multigrid.py:51-55`,
  prolongation / restriction `multigrid.py:91-130`, the V-cycle with a dense
  coarse solve `multigrid.py:326-350`; preconditioned CG `krylov.py:69-123`.

Parity pin: `tests/test_oracle.py` checks this oracle against golden vectors
produced by the reference itself (`tests/golden/make_golden.py`,
`tests/golden/make_golden_mg.py`).
"""

from __future__ import annotations

import itertools

import numpy as np
from numpy.polynomial import legendre as npleg


# ---------------------------------------------------------------- 1D setup --
def gl_nodes(k):
    """`polybasis.py:48-67`."""
    if k == 1:
        return np.array([0.0, 1.0])
    c = np.zeros(k + 1)
    c[k] = 1.0
    dc = npleg.legder(c)
    x = np.real(npleg.legroots(dc))
    x = x - npleg.legval(x, dc) / npleg.legval(x, npleg.legder(dc))
    x.sort()
    return (np.concatenate(([-1.0], x, [1.0])) + 1.0) / 2.0


def lagrange(nodes, x):
    """values and derivatives of the Lagrange basis (`polybasis.py:90-133`)."""
    x = np.atleast_1d(np.asarray(x, dtype=float))
    n = len(nodes)
    val = np.empty((n, len(x)))
    der = np.zeros((n, len(x)))
    for i in range(n):
        num = np.ones_like(x)
        den = 1.0
        for j in range(n):
            if j != i:
                num *= x - nodes[j]
                den *= nodes[i] - nodes[j]
        val[i] = num / den
        acc = np.zeros_like(x)
        for j in range(n):
            if j == i:
                continue
            term = np.ones_like(x)
            for l in range(n):
                if l != i and l != j:
                    term *= x - nodes[l]
            acc += term
        der[i] = acc / den
    return val, der


class Setup1D:
    """All 1D matrices of a uniform level with cell length h."""

    def __init__(self, k, h, gamma_hat=1.0):
        self.k, self.n, self.h, self.gamma_hat = k, k + 1, h, gamma_hat
        nodes = gl_nodes(k)
        xq, wq = npleg.leggauss(k + 1)
        xq, wq = (xq + 1.0) / 2.0, wq / 2.0
        v, g = lagrange(nodes, xq)
        bv, bg = lagrange(nodes, np.array([0.0, 1.0]))
        self.bv, self.bg = bv.T.copy(), bg.T.copy()          # (2, n)
        self.mass = h * (v * wq) @ v.T                        # polybasis.py:240-244
        self.bulk = (1.0 / h) * (g * wq) @ g.T
        self.ge = gamma_hat * k * (k + 1) * (2.0 / h)         # polybasis.py:170-174

    def nitsche(self, p, boundary):
        """`polybasis.py:216-237`."""
        eta = 1.0 if boundary else 0.5
        s = -1.0 if p == 0 else 1.0
        g = s * (eta / self.h) * np.outer(self.bv[p], self.bg[p])
        return eta * self.ge * np.outer(self.bv[p], self.bv[p]) - g - g.T

    def cell_stiffness(self, digit):
        return self.bulk + self.nitsche(0, bool(digit & 1)) + self.nitsche(1, bool(digit & 2))

    def coupling(self):
        """a_pm, rows test on the left cell, cols trial on the right cell."""
        h = self.h
        return (-0.5 * self.ge) * np.outer(self.bv[1], self.bv[0]) \
            - (0.5 / h) * np.outer(self.bv[1], self.bg[0]) \
            + (0.5 / h) * np.outer(self.bg[1], self.bv[0])

    def patch_matrices(self, digit):
        n = self.n
        a = np.zeros((2 * n, 2 * n))
        m = np.zeros((2 * n, 2 * n))
        a[:n, :n] = self.bulk + self.nitsche(0, bool(digit & 1)) + self.nitsche(1, False)
        a[n:, n:] = self.bulk + self.nitsche(0, False) + self.nitsche(1, bool(digit & 2))
        a[:n, n:] = self.coupling()
        a[n:, :n] = self.coupling().T
        m[:n, :n] = self.mass
        m[n:, n:] = self.mass
        return a, m


def geneig(a, m):
    """Cholesky reduction + eigh (`polybasis.py:313-341`)."""
    import scipy.linalg as sla

    lc = np.linalg.cholesky(m)
    c = sla.solve_triangular(lc, a, lower=True)
    c = sla.solve_triangular(lc, c.T, lower=True)
    lam, v = np.linalg.eigh(0.5 * (c + c.T))
    return sla.solve_triangular(lc.T, v, lower=False), lam


# ---------------------------------------------------------------- level ----
def _along(x, mat, axis):
    """out[.., i, ..] = sum_k mat[i, k] x[.., k, ..] along `axis`."""
    return np.moveaxis(np.tensordot(mat, x, axes=([1], [axis])), 0, axis)


class OracleLevel:
    """Uniform Cartesian box: dims[t] cells along direction t+1, length h."""

    def __init__(self, dims, k, h=None, gamma_hat=1.0):
        self.dims = tuple(int(v) for v in dims)
        self.d = len(self.dims)
        self.k, self.n = k, k + 1
        self.h = 1.0 / self.dims[0] if h is None else h
        self.s = Setup1D(k, self.h, gamma_hat)
        self.ncells = int(np.prod(self.dims))
        self.ndofs = self.ncells * self.n ** self.d

    # grid view: axes (c_d .. c_1, i_d .. i_1)
    def grid(self, x):
        return x.reshape(self.dims[::-1] + (self.n,) * self.d)

    def cell_axis(self, t):
        return self.d - 1 - t

    def node_axis(self, t):
        return 2 * self.d - 1 - t

    # -------------------------------------------------------------- operator
    def apply(self, x):
        """v = A x, Kronecker-sum form."""
        X = self.grid(np.asarray(x, dtype=float))
        V = np.zeros_like(X)
        s = self.s
        apm = s.coupling()
        for t in range(self.d):
            ca, na = self.cell_axis(t), self.node_axis(t)
            nt = self.dims[t]
            G = np.empty_like(X)
            for c in range(nt):
                digit = (1 if c == 0 else 0) | (2 if c == nt - 1 else 0)
                sl = [slice(None)] * X.ndim
                sl[ca] = c
                xs = X[tuple(sl)]
                g = _along(xs, s.cell_stiffness(digit), na - 1)
                if c + 1 < nt:
                    sl2 = list(sl)
                    sl2[ca] = c + 1
                    g = g + _along(X[tuple(sl2)], apm, na - 1)
                if c > 0:
                    sl2 = list(sl)
                    sl2[ca] = c - 1
                    g = g + _along(X[tuple(sl2)], apm.T, na - 1)
                G[tuple(sl)] = g
            for u in range(self.d):
                if u != t:
                    G = _along(G, s.mass, self.node_axis(u))
            V += G
        return V.reshape(-1)

    def residual(self, x, b):
        return np.asarray(b, dtype=float) - self.apply(x)

    def dense(self):
        """Dense level matrix from unit vectors of `apply` (tiny levels)."""
        if self.ndofs > 6000:
            raise ValueError("dense oracle limited to 6000 dofs")
        e = np.zeros(self.ndofs)
        a = np.empty((self.ndofs, self.ndofs))
        for j in range(self.ndofs):
            e[j] = 1.0
            a[:, j] = self.apply(e)
            e[j] = 0.0
        return a

    # ------------------------------------------------------------ subdomains
    def cell_digits(self):
        """(ncells, d) digits, cell id order."""
        pos = np.stack(np.unravel_index(np.arange(self.ncells), self.dims[::-1])[::-1], axis=1)
        last = np.array(self.dims) - 1
        return (pos == 0).astype(int) + 2 * (pos == last[None, :]).astype(int)

    def patch_vertices(self):
        """(P, d) interior vertices, v_1 fastest (`mesh.py:307-310`)."""
        if min(self.dims) < 2:
            return np.empty((0, self.d), dtype=np.int64)
        axes = [np.arange(1, v) for v in self.dims]
        g = np.meshgrid(*axes[::-1], indexing="ij")
        return np.stack([a.ravel() for a in g[::-1]], axis=-1).astype(np.int64)

    def patch_digits(self, v):
        last = np.array(self.dims) - 1
        return (v == 1).astype(int) + 2 * (v == last[None, :]).astype(int)

    def patch_map(self, v):
        """(P, m^d) global dof indices, patch-local canonical order
        (`fastdiag.py:546-582`)."""
        d, n = self.d, self.n
        m = 2 * n
        strides = np.cumprod((1,) + self.dims[:-1]).astype(np.int64)
        q = np.indices((m,) * d).reshape(d, -1)[::-1]          # q[t] = digit of direction t
        block = q // n
        within = q % n
        off = (within * (n ** np.arange(d))[:, None]).sum(axis=0)
        cell = ((v[:, :, None] - 1 + block[None, :, :]) * strides[None, :, None]).sum(axis=1)
        return cell * n ** d + off[None, :]

    def patch_colors(self, v):
        """`mesh.py:360-375`."""
        par = ((v % 2) * (2 ** np.arange(self.d))[None, :]).sum(axis=1)
        return par * 2 + (v // 2).sum(axis=1) % 2

    def _fdm(self, R, digits, m, kind):
        """Y = Z Lambda^-1 Z^T R per subdomain (rows of R, canonical m^d)."""
        s = self.s
        d = self.d
        out = np.empty_like(R)
        pairs = {}
        for dg in range(4):
            if kind == "cell":
                pairs[dg] = geneig(s.cell_stiffness(dg), s.mass)
            else:
                pairs[dg] = geneig(*s.patch_matrices(dg))
        codes = (digits * (4 ** np.arange(d))[None, :]).sum(axis=1)
        for code in np.unique(codes):
            sel = np.nonzero(codes == code)[0]
            dg = digits[sel[0]]
            Y = R[sel].reshape((len(sel),) + (m,) * d)
            lam_sum = 0.0
            for t in range(d):
                z, lam = pairs[dg[t]]
                Y = _along(Y, z.T, d - t)
                shape = [1] * d
                shape[d - 1 - t] = m
                lam_sum = lam_sum + lam.reshape(shape)
            if np.any(lam_sum <= 0):
                raise ValueError("nonpositive Kronecker-sum eigenvalue")
            Y = Y / lam_sum[None]
            for t in range(d - 1, -1, -1):
                z, _ = pairs[dg[t]]
                Y = _along(Y, z, d - t)
            out[sel] = Y.reshape(len(sel), -1)
        return out

    def cell_solve(self, x, r, omega, cells=None):
        """x[cells] += omega A_c^-1 r_c (`fastdiag.py:457-496`)."""
        nd = self.n ** self.d
        cells = np.arange(self.ncells) if cells is None else np.asarray(cells)
        R = np.asarray(r).reshape(-1, nd)[cells]
        Y = self._fdm(R, self.cell_digits()[cells], self.n, "cell")
        x.reshape(-1, nd)[cells] += omega * Y

    def patch_solve(self, x, r, omega, patches=None, safe=False):
        """x[R_j] += omega A_j^-1 R_j r (`fastdiag.py:602-628`)."""
        v = self.patch_vertices()
        if patches is not None:
            v = v[np.asarray(patches)]
        if len(v) == 0:
            return
        gi = self.patch_map(v)
        Y = self._fdm(np.asarray(r)[gi], self.patch_digits(v), 2 * self.n, "patch")
        if safe:
            np.add.at(x, gi.ravel(), (omega * Y).ravel())
        else:
            x[gi] += omega * Y

    # ----------------------------------------------------------- smoothing
    def colours(self, kind):
        if kind == "acs":
            return [np.arange(self.ncells)]
        if kind == "mcs":
            par = np.indices(self.dims[::-1]).sum(axis=0).ravel() % 2
            ids = np.arange(self.ncells)
            return [s for s in (ids[par == 0], ids[par == 1]) if len(s)]
        v = self.patch_vertices()
        col = self.patch_colors(v)
        ids = np.arange(len(v))
        return [s for s in (ids[col == c] for c in range(2 ** (self.d + 1))) if len(s)]

    def smooth(self, kind, omega, x, b, reverse=False):
        """One step (`smoothers.py:131-166`); returns a new vector."""
        x = np.array(x, dtype=float, copy=True)
        cols = self.colours(kind)
        solve = self.cell_solve if kind in ("acs", "mcs") else self.patch_solve
        if kind in ("acs", "avs"):
            r = self.residual(x, b)
            for c in cols:
                solve(x, r, omega, c)
        else:
            order = cols[::-1] if reverse else cols
            for c in order:
                r = self.residual(x, b)
                solve(x, r, omega, c)
        return x


def seeded_inputs(ndofs, seed=0):
    """b ~ U[-1,1] from seed, x0 ~ U[-1,1] from seed+1."""
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, ndofs)
    x0 = np.random.default_rng(seed + 1).uniform(-1.0, 1.0, ndofs)
    return x0, b


# ------------------------------------------------- multigrid --
def embeddings(k):
    """E^s[i, j] = phi_j((x_i + s) / 2), s = 0, 1 (`multigrid.py:51-55`)."""
    nodes = gl_nodes(k)
    return lagrange(nodes, nodes / 2.0)[0].T.copy(), lagrange(nodes, (nodes + 1.0) / 2.0)[0].T.copy()


def _children(dims, n):
    """(child bits s_t per direction, fine-grid slice) for the 2^d children."""
    d = len(dims)
    for s in itertools.product((0, 1), repeat=d):
        sl = [slice(None)] * (2 * d)
        for t in range(d):
            sl[d - 1 - t] = slice(s[t], None, 2)   # cell axis of direction t
        yield s, tuple(sl)


def prolongate(dims, k, xc):
    """Fine cell 2c+s gets (E^{s_d} x .. x E^{s_1}) x_c (`multigrid.py:91-108`);
    `dims` are the coarse cells per direction."""
    d, n = len(dims), k + 1
    e = embeddings(k)
    X = np.asarray(xc, dtype=float).reshape(tuple(dims[::-1]) + (n,) * d)
    F = np.empty(tuple(2 * v for v in dims[::-1]) + (n,) * d)
    for s, sl in _children(dims, n):
        Y = X
        for t in range(d):
            Y = _along(Y, e[s[t]], 2 * d - 1 - t)
        F[sl] = Y
    return F.reshape(-1)


def restrict(dims, k, xf):
    """Adjoint of `prolongate` (`multigrid.py:110-130`)."""
    d, n = len(dims), k + 1
    e = embeddings(k)
    F = np.asarray(xf, dtype=float).reshape(tuple(2 * v for v in dims[::-1]) + (n,) * d)
    X = np.zeros(tuple(dims[::-1]) + (n,) * d)
    for s, sl in _children(dims, n):
        Y = F[sl]
        for t in range(d):
            Y = _along(Y, e[s[t]].T, 2 * d - 1 - t)
        X += Y
    return X.reshape(-1)


class OracleVCycle:
    """V-cycle over cube levels coarse*2^l (`multigrid.py:296-350`) with a
    dense direct coarse solve (`multigrid.py:170-176`)."""

    def __init__(self, d, coarse, levels, k, kind, omega, m_pre=1, m_post=1,
                 symmetrize=False):
        self.levels = [OracleLevel((coarse * 2 ** l,) * d, k) for l in range(levels + 1)]
        self.k, self.kind, self.omega = k, kind, omega
        self.m_pre, self.m_post, self.sym = m_pre, m_post, symmetrize
        self._a0 = self.levels[0].dense()

    def vcycle(self, ell, x, b):
        if ell == 0:
            return np.linalg.solve(self._a0, b)
        lv = self.levels[ell]
        for _ in range(self.m_pre):
            x = lv.smooth(self.kind, self.omega, x, b)
        bc = restrict(self.levels[ell - 1].dims, self.k, lv.residual(x, b))
        xc = self.vcycle(ell - 1, np.zeros_like(bc), bc)
        x = x + prolongate(self.levels[ell - 1].dims, self.k, xc)
        for _ in range(self.m_post):
            x = lv.smooth(self.kind, self.omega, x, b, reverse=self.sym)
        return x

    def apply(self, b):
        return self.vcycle(len(self.levels) - 1, np.zeros_like(b), b)


def pcg(apply_op, b, precond, delta_red=1e-8, max_it=200):
    """Preconditioned CG (`krylov.py:69-123`): returns (x, residual history)."""
    x = np.zeros_like(b)
    r = b.copy()
    hist = [np.linalg.norm(r)]
    if hist[0] == 0.0:
        return x, hist
    z = precond(r)
    p = z.copy()
    rz = r @ z
    for _ in range(max_it):
        ap = apply_op(p)
        alpha = rz / (p @ ap)
        x += alpha * p
        r -= alpha * ap
        hist.append(np.linalg.norm(r))
        if hist[-1] <= delta_red * hist[0]:
            break
        z = precond(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, hist
