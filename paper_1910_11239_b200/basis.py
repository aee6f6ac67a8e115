"""Host-side 1D setup: Gauss-Lobatto Lagrange basis, Gauss rule, the
univariate SIPG factors and the symmetric-definite generalised eigenpairs.

This is the "tiny 1D eigenproblem stays on the host" part of the north star:
everything here is O(k^3) numpy work done once per level, whose outputs are
uploaded to the device as small tables (see `tables.py`).  The math follows
the reference's polybasis module; each function cites the lines it restates:

- GL nodes: endpoints plus the roots of P_k' with one Newton polish
  (`pkg/src/dgmg/polybasis.py:48-67`);
- Gauss rule with k+1 points on [0,1] (`polybasis.py:82-87`, `151-153`);
- Lagrange values / derivatives by direct products (`polybasis.py:90-133`);
- cell factor A = L + N_0 + N_1 with trace weight eta (`polybasis.py:224-259`);
- patch factor [[A+, a_pm], [a_pm^T, A-]] (`polybasis.py:262-302`);
- Cholesky-reduced eigenproblem, Z^T A Z = diag(lam), Z^T M Z = I
  (`polybasis.py:313-341`).

The operations are ordered like the reference's so that the uploaded tables
agree with it to the last bit on the same numpy/LAPACK build (tests pin this).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from numpy.polynomial import legendre as _leg

__all__ = [
    "Basis1D",
    "MassNotSPDError",
    "EigenSolveError",
    "gl_nodes",
    "gauss_rule",
    "lagrange_table",
    "lagrange_deriv_table",
    "sipg_penalty",
    "cell_factors",
    "patch_factors",
    "sym_eig",
]


class MassNotSPDError(np.linalg.LinAlgError):
    """Mass matrix without a Cholesky factor (`polybasis.py:40-41`)."""


class EigenSolveError(np.linalg.LinAlgError):
    """Symmetric eigensolver failure (`polybasis.py:44-45`)."""


def gl_nodes(k: int) -> np.ndarray:
    """k+1 Gauss-Lobatto points on [0,1] (`polybasis.py:48-67`)."""
    if k < 1:
        raise ValueError("polynomial degree must be >= 1")
    if k == 1:
        return np.array([0.0, 1.0])
    pk = np.zeros(k + 1)
    pk[k] = 1.0
    d1 = _leg.legder(pk)
    inner = np.real(_leg.legroots(d1))
    d2 = _leg.legder(d1)
    inner = inner - _leg.legval(inner, d1) / _leg.legval(inner, d2)
    inner.sort()
    return (np.concatenate(([-1.0], inner, [1.0])) + 1.0) / 2.0


def gauss_rule(npts: int) -> tuple[np.ndarray, np.ndarray]:
    """Gauss-Legendre points/weights on [0,1] (`polybasis.py:82-87`)."""
    if npts < 1:
        raise ValueError("quadrature point count must be >= 1")
    x, w = _leg.leggauss(npts)
    return (x + 1.0) / 2.0, w / 2.0


def lagrange_table(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """phi_i(x_q), shape (len(nodes), len(x)) (`polybasis.py:90-109`)."""
    nodes = np.asarray(nodes, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    n = len(nodes)
    out = np.empty((n, len(x)))
    for i in range(n):
        num = np.ones_like(x)
        den = 1.0
        for j in range(n):
            if j != i:
                num *= x - nodes[j]
                den *= nodes[i] - nodes[j]
        out[i] = num / den
    return out


def lagrange_deriv_table(nodes: np.ndarray, x: np.ndarray) -> np.ndarray:
    """phi_i'(x_q) by the product rule (`polybasis.py:111-133`)."""
    nodes = np.asarray(nodes, dtype=float)
    x = np.atleast_1d(np.asarray(x, dtype=float))
    n = len(nodes)
    out = np.zeros((n, len(x)))
    for i in range(n):
        den = 1.0
        for j in range(n):
            if j != i:
                den *= nodes[i] - nodes[j]
        acc = np.zeros_like(x)
        for j in range(n):
            if j == i:
                continue
            term = np.ones_like(x)
            for l in range(n):
                if l != i and l != j:
                    term *= x - nodes[l]
            acc += term
        out[i] = acc / den
    return out


@dataclass(frozen=True)
class Basis1D:
    """Degree-k Lagrange basis on GL nodes with k+1 Gauss points
    (`polybasis.py:136-167`).  `bv[p]`, `bg[p]` are values / derivatives of
    all basis functions at x = p for p in {0, 1}."""

    degree: int
    nodes: np.ndarray
    qpts: np.ndarray
    qwts: np.ndarray
    values: np.ndarray   # (n, nq)
    grads: np.ndarray    # (n, nq)
    bv: np.ndarray       # (2, n)
    bg: np.ndarray       # (2, n)

    @classmethod
    def make(cls, k: int, n_q: int | None = None) -> "Basis1D":
        nodes = gl_nodes(k)
        qp, qw = gauss_rule(k + 1 if n_q is None else n_q)
        ends = np.array([0.0, 1.0])
        return cls(degree=k, nodes=nodes, qpts=qp, qwts=qw,
                   values=lagrange_table(nodes, qp),
                   grads=lagrange_deriv_table(nodes, qp),
                   bv=lagrange_table(nodes, ends).T.copy(),
                   bg=lagrange_deriv_table(nodes, ends).T.copy())

    @property
    def n(self) -> int:
        return self.degree + 1


def sipg_penalty(gamma_hat: float, k: int, h_plus: float, h_minus: float) -> float:
    """gamma_hat k(k+1)(1/h+ + 1/h-) (`polybasis.py:170-174`)."""
    if h_plus <= 0.0 or h_minus <= 0.0:
        raise ValueError("cell lengths must be positive")
    return gamma_hat * k * (k + 1) * (1.0 / h_plus + 1.0 / h_minus)


def _nitsche(basis: Basis1D, h: float, p: int, boundary: bool,
             h_nb: float | None, gamma_hat: float) -> np.ndarray:
    """eta*gamma_e*bv_p bv_p^T - G - G^T with G = s_p (eta/h) bv_p bg_p^T
    (`polybasis.py:216-237`)."""
    eta = 1.0 if boundary else 0.5
    hn = h if boundary or h_nb is None else h_nb
    ge = sipg_penalty(gamma_hat, basis.degree, h, hn)
    sgn = -1.0 if p == 0 else 1.0
    bv = basis.bv[p]
    g = sgn * (eta / h) * np.outer(bv, basis.bg[p])
    return eta * ge * np.outer(bv, bv) - g - g.T


def _mass_bulk(basis: Basis1D, h: float) -> tuple[np.ndarray, np.ndarray]:
    """h * V W V^T and (1/h) G W G^T (`polybasis.py:240-244`)."""
    w = basis.qwts
    mass = h * (basis.values * w) @ basis.values.T
    bulk = (1.0 / h) * (basis.grads * w) @ basis.grads.T
    return mass, bulk


def cell_factors(basis: Basis1D, h: float, left_bnd: bool, right_bnd: bool,
                 gamma_hat: float = 1.0, h_left: float | None = None,
                 h_right: float | None = None) -> tuple[np.ndarray, np.ndarray]:
    """(mass, stiffness) of one interval (`polybasis.py:247-259`)."""
    if h <= 0.0:
        raise ValueError("interval length must be positive")
    mass, bulk = _mass_bulk(basis, h)
    n0 = _nitsche(basis, h, 0, left_bnd, h_left, gamma_hat)
    n1 = _nitsche(basis, h, 1, right_bnd, h_right, gamma_hat)
    return mass, bulk + n0 + n1


def interface_block(basis: Basis1D, h_plus: float, h_minus: float,
                    gamma_hat: float = 1.0) -> np.ndarray:
    """Rank-2 coupling a_pm (rows: test on the left interval I+, cols: trial
    on the right interval I-) (`polybasis.py:278-284`)."""
    ge = sipg_penalty(gamma_hat, basis.degree, h_plus, h_minus)
    bv0, bv1 = basis.bv
    bg0, bg1 = basis.bg
    return (-0.5 * ge) * np.outer(bv1, bv0) \
        - (0.5 / h_minus) * np.outer(bv1, bg0) \
        + (0.5 / h_plus) * np.outer(bg1, bv0)


def patch_factors(basis: Basis1D, h_plus: float, h_minus: float,
                  left_bnd: bool, right_bnd: bool,
                  gamma_hat: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """(mass, stiffness) of a two-interval vertex-patch direction, blocked
    [I+, I-] (`polybasis.py:262-302`)."""
    if h_plus <= 0.0 or h_minus <= 0.0:
        raise ValueError("interval lengths must be positive")
    mp, ap = cell_factors(basis, h_plus, left_bnd, False, gamma_hat,
                          h_right=h_minus)
    mm, am = cell_factors(basis, h_minus, False, right_bnd, gamma_hat,
                          h_left=h_plus)
    apm = interface_block(basis, h_plus, h_minus, gamma_hat)
    n = basis.n
    mass = np.zeros((2 * n, 2 * n))
    mass[:n, :n] = mp
    mass[n:, n:] = mm
    stiff = np.zeros((2 * n, 2 * n))
    stiff[:n, :n] = ap
    stiff[n:, n:] = am
    stiff[:n, n:] = apm
    stiff[n:, :n] = apm.T
    return mass, stiff


def sym_eig(a: np.ndarray, m: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(Z, lam) with Z^T A Z = diag(lam) ascending, Z^T M Z = I, by Cholesky
    reduction (`polybasis.py:313-341`)."""
    import scipy.linalg as sla

    a = np.asarray(a, dtype=float)
    m = np.asarray(m, dtype=float)
    scale = np.linalg.norm(a, ord=np.inf)
    if scale > 0 and np.linalg.norm(a - a.T, ord=np.inf) > 1e-12 * scale:
        raise ValueError("stiffness matrix is not symmetric")
    try:
        lc = np.linalg.cholesky(m)
    except np.linalg.LinAlgError as exc:
        raise MassNotSPDError("mass not SPD") from exc
    c = sla.solve_triangular(lc, a, lower=True)
    c = sla.solve_triangular(lc, c.T, lower=True)
    c = 0.5 * (c + c.T)
    try:
        lam, v = np.linalg.eigh(c)
    except np.linalg.LinAlgError as exc:
        raise EigenSolveError("symmetric eigensolver did not converge") from exc
    z = sla.solve_triangular(lc.T, v, lower=False)
    return z, lam
