"""Per-level device tables from the 1D host setup.

On a uniform Cartesian level every 1D object depends only on the boundary
pattern of one direction, the *digit* (bit 0: left face on the boundary,
bit 1: right face on the boundary; `fastdiag.py:349-369`, `535-566`), so a
level needs at most four 1D problems per kind.  This module builds:

- operator: the cell mass M, the cell stiffness A_diag(digit) (the diagonal
  blocks of the block-tridiagonal 1D SIPG matrix, `polybasis.py:247-259`),
  and the rank-2 coupling a_pm in factored form (alpha, beta, beta', bg0,
  bg1; `polybasis.py:278-284`), valid because GL bases have
  bv0 = e_0, bv1 = e_(n-1) exactly (asserted);
- cell FDM: Z, Z^T per digit and 1/Lambda-sum per class code
  (`fastdiag.py:89-100`, `136-154`), canonical layout;
- patch FDM: the same for the 2n x 2n two-cell factors (`fastdiag.py:157-177`).

Class code = sum_t digit_t 4^t; the singular check of `_inverse_sum_reversed`
(`fastdiag.py:98-99`) runs over the classes the level actually has.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .basis import Basis1D, cell_factors, patch_factors, sipg_penalty, sym_eig


class SingularLocalSolverError(ValueError):
    """A Kronecker-sum eigenvalue is not positive (`fastdiag.py:50-51`)."""


def cell_digits(n_t: int) -> list[int]:
    """Digits that occur for cells along a direction with n_t cells."""
    if n_t == 1:
        return [3]
    return ([0] if n_t >= 3 else []) + [1, 2]


def patch_digits(n_t: int) -> list[int]:
    """Digits that occur for interior vertices v in [1, n_t-1]."""
    if n_t < 2:
        return []
    if n_t == 2:
        return [3]
    return ([0] if n_t >= 4 else []) + [1, 2]


def inverse_sum(lams: list[np.ndarray]) -> np.ndarray:
    """1/(lam_1[i_1] + ... + lam_d[i_d]) in canonical layout (i_d slowest);
    sums in direction order like `fastdiag.py:89-100`."""
    d = len(lams)
    total = None
    for t, lam in enumerate(lams):
        shape = [1] * d
        shape[d - 1 - t] = lam.size
        arr = lam.reshape(shape)
        total = arr if total is None else total + arr
    if np.any(total <= 0.0):
        raise SingularLocalSolverError("nonpositive Kronecker-sum eigenvalue")
    return 1.0 / total


@dataclass
class LevelTables:
    dim: int
    degree: int
    h: float
    gamma_hat: float
    mass: np.ndarray          # (n, n)
    adiag: np.ndarray         # (4, n, n)
    bg: np.ndarray            # (2, n)
    alpha: float
    beta: float
    betap: float
    cell_z: np.ndarray        # (4, n, n)
    cell_lam: np.ndarray      # (4, n)
    cell_invsum: np.ndarray   # (4^d, n^d)
    patch_z: np.ndarray | None
    patch_lam: np.ndarray | None
    patch_invsum: np.ndarray | None

    @property
    def n(self) -> int:
        return self.degree + 1


def _classes(dims, digits_of):
    per = [digits_of(n_t) for n_t in dims]
    codes = [0]
    digs = [[]]
    for t, opts in enumerate(per):
        codes = [c + dg * 4 ** t for c in codes for dg in opts]
        digs = [dl + [dg] for dl in digs for dg in opts]
    return list(zip(codes, digs))


def build_tables(basis: Basis1D, h: float, dims: tuple[int, ...],
                 gamma_hat: float = 1.0, with_patches: bool = True) -> LevelTables:
    d = len(dims)
    k = basis.degree
    n = basis.n
    if not (np.array_equal(basis.bv[0], np.eye(n)[0])
            and np.array_equal(basis.bv[1], np.eye(n)[n - 1])):
        raise ValueError("device operator needs a nodal basis with end nodes at 0 and 1")
    mass = None
    adiag = np.empty((4, n, n))
    cz = np.empty((4, n, n))
    clam = np.empty((4, n))
    for digit in range(4):
        m_, a_ = cell_factors(basis, h, bool(digit & 1), bool(digit & 2), gamma_hat)
        mass = m_ if mass is None else mass
        adiag[digit] = a_
        cz[digit], clam[digit] = sym_eig(a_, m_)
    ge = sipg_penalty(gamma_hat, k, h, h)
    cinv = np.zeros((4 ** d, n ** d))
    for code, digs in _classes(dims, cell_digits):
        cinv[code] = inverse_sum([clam[dg] for dg in digs]).ravel()

    pz = plam = pinv = None
    if with_patches and min(dims) >= 2:
        m = 2 * n
        pz = np.empty((4, m, m))
        plam = np.empty((4, m))
        for digit in range(4):
            pm, pa = patch_factors(basis, h, h, bool(digit & 1), bool(digit & 2), gamma_hat)
            pz[digit], plam[digit] = sym_eig(pa, pm)
        pinv = np.zeros((4 ** d, m ** d))
        for code, digs in _classes(dims, patch_digits):
            pinv[code] = inverse_sum([plam[dg] for dg in digs]).ravel()

    return LevelTables(dim=d, degree=k, h=h, gamma_hat=gamma_hat, mass=mass,
                       adiag=adiag, bg=basis.bg.copy(), alpha=-0.5 * ge,
                       beta=-0.5 / h, betap=0.5 / h, cell_z=cz, cell_lam=clam,
                       cell_invsum=cinv, patch_z=pz, patch_lam=plam,
                       patch_invsum=pinv)


# ---------------------------------------------------------------------------
# device packing: even/odd (centro-symmetric) factorisation of the interior
# digit.  On an interior direction the 1D pencil is symmetric about the cell
# (patch) midpoint, so the eigenvectors are even or odd and M, A_diag are
# centro-symmetric: each m x m contraction splits into two (m/2) x (m/2) ones
# on u = v_i + v_{m-1-i}, w = v_i - v_{m-1-i} (half the FMAs).  The interior
# eigenpairs are reordered even-first (the FDM inverse is invariant under a
# consistent permutation of eigenpairs and 1/Lambda-sum).
# ---------------------------------------------------------------------------
EO_TOL = 1e-12


def _parity(z: np.ndarray):
    """0/1 parity of each column of z, or None if not exactly symmetric."""
    par = []
    scale = np.abs(z).max()
    for j in range(z.shape[1]):
        ev = np.abs(z[:, j] - z[::-1, j]).max()
        od = np.abs(z[:, j] + z[::-1, j]).max()
        if min(ev, od) > EO_TOL * scale:
            return None
        par.append(0 if ev <= od else 1)
    par = np.array(par)
    if z.shape[0] % 2 or par.sum() * 2 != z.shape[0]:
        return None
    return par


def _eo_fdm(z: np.ndarray, lam: np.ndarray):
    """(permuted z, permuted lam, [fwdE, fwdO, bwdE, bwdO]) or None."""
    par = _parity(z)
    if par is None:
        return None
    perm = np.concatenate([np.nonzero(par == 0)[0], np.nonzero(par == 1)[0]])
    zp = z[:, perm]
    lp = lam[perm]
    h = z.shape[0] // 2
    top = zp[:h]
    halves = np.stack([top[:, :h], top[:, h:], top[:, :h].T, top[:, h:].T])
    return zp, lp, np.ascontiguousarray(halves)


def _cs_halves(a: np.ndarray):
    """k-outer (transposed) P, Q of a centro-symmetric matrix, or None."""
    m = a.shape[0]
    if m % 2 or np.abs(a - a[::-1, ::-1]).max() > EO_TOL * np.abs(a).max():
        return None
    h = m // 2
    p = 0.5 * (a[:h, :h] + a[:h, ::-1][:, :h])
    q = 0.5 * (a[:h, :h] - a[:h, ::-1][:, :h])
    return np.stack([p.T, q.T])


@dataclass
class DeviceTables:
    cell_z: np.ndarray
    cell_invsum: np.ndarray
    cell_eo: np.ndarray | None
    patch_z: np.ndarray | None
    patch_invsum: np.ndarray | None
    patch_eo: np.ndarray | None
    res_eo: np.ndarray | None


def device_tables(t: LevelTables, dims: tuple[int, ...], use_eo: bool = True) -> DeviceTables:
    d = t.dim
    cz, clam, cinv, ceo = t.cell_z.copy(), t.cell_lam.copy(), t.cell_invsum, None
    if use_eo:
        r = _eo_fdm(t.cell_z[0], t.cell_lam[0])
        if r is not None:
            cz[0], clam[0], ceo = r
            cinv = np.zeros_like(t.cell_invsum)
            for code, digs in _classes(dims, cell_digits):
                cinv[code] = inverse_sum([clam[dg] for dg in digs]).ravel()
    pz = pinv = peo = None
    if t.patch_z is not None:
        pz, plam, pinv = t.patch_z.copy(), t.patch_lam.copy(), t.patch_invsum
        if use_eo:
            r = _eo_fdm(t.patch_z[0], t.patch_lam[0])
            if r is not None:
                pz[0], plam[0], peo = r
                pinv = np.zeros_like(t.patch_invsum)
                for code, digs in _classes(dims, patch_digits):
                    pinv[code] = inverse_sum([plam[dg] for dg in digs]).ravel()
    reo = None
    if use_eo:
        mh, ah = _cs_halves(t.mass), _cs_halves(t.adiag[0])
        if mh is not None and ah is not None:
            reo = np.ascontiguousarray(np.concatenate([mh, ah]))
    return DeviceTables(cz, cinv, ceo, pz, pinv, peo, reo)
