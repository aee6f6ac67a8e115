"""Work accounting with the reference's conventions (`pkg/src/dgmg/flops.py`).

`FlopCounter` has the reference's interface (`flops.py:22-47`) so callers such
as the complexity probe keep working; the counts are the reference's analytic
formulas (1 op per add/mul, FMAs not collapsed), not what the GPU executes.
`step_work()` is the SURVEY 8(d) work model used for the roofline: minimal
Kronecker-form residual flops plus the exact local-solver count, FMA = 2.
"""

from __future__ import annotations

EIG_MODEL_FLOPS_N3 = 9.0


class FlopCounter:
    def __init__(self):
        self.counts: dict[str, float] = {}

    def add(self, kernel: str, flops: float) -> None:
        self.counts[kernel] = self.counts.get(kernel, 0.0) + float(flops)

    def get(self, kernel: str) -> float:
        return self.counts.get(kernel, 0.0)

    def total(self) -> float:
        return float(sum(self.counts.values()))

    def snapshot(self) -> dict[str, float]:
        return dict(self.counts)

    def reset(self) -> None:
        self.counts.clear()


def contraction_flops(batch: int, out_elems: int, inner: int) -> float:
    """`flops.py:50-52`."""
    return float(batch) * out_elems * (2 * inner - 1)


def generalized_eig_flops(n: int) -> float:
    """`flops.py:72-79`."""
    return n ** 3 / 3.0 + 2.0 * n ** 3 + 0.5 * n ** 3 + EIG_MODEL_FLOPS_N3 * n ** 3


def univariate_assembly_flops(n: int, q: int) -> float:
    """`flops.py:82-84`."""
    return 2.0 * n * n * (2 * q - 1) + 4.0 * (3 * n * n)


def local_solver_setup_flops(d: int, k: int, kind: str = "cell") -> float:
    """`flops.py:86-92`."""
    n = k + 1 if kind == "cell" else 2 * (k + 1)
    per_dir = univariate_assembly_flops(n, k + 1) + generalized_eig_flops(n)
    return d * per_dir + d * n ** d


def local_solver_apply_flops(d: int, m: int) -> float:
    """`flops.py:95-97`."""
    return 2.0 * d * contraction_flops(1, m ** d, m) + m ** d


def operator_apply_flops(d: int, n: int, q: int, dims: tuple[int, ...]) -> float:
    """Reference count of one Cartesian `apply_operator` (volume
    `dgop.py:443-481` + faces `dgop.py:583-759`) on a box."""
    ncells = 1
    for v in dims:
        ncells *= v
    Q = q ** d
    stages = (d - 1) + d * (d + 1) // 2
    flops = ncells * Q * d + 2 * stages * contraction_flops(ncells, Q, n) + ncells * Q
    qf = q ** (d - 1) if d > 1 else 1
    for tau in range(d):
        trans = ncells // dims[tau]
        nf = (dims[tau] - 1) * trans
        if nf > 0:
            per_side = 2 * contraction_flops(nf, n ** (d - 1), n)
            if d > 1:
                per_side += (2 + d) * contraction_flops(nf, qf, n)
            flops += nf * qf * 8 + 4 * per_side
        for _ in range(2):
            per_side = 2 * contraction_flops(trans, n ** (d - 1), n)
            if d > 1:
                per_side += (2 + d) * contraction_flops(trans, qf, n)
            flops += trans * qf * 5 + 2 * per_side
    return float(flops)


def residual_flops_min(d: int, n: int, ncells: int) -> float:
    """Minimal Kronecker-form residual count:
    n_cells (2(3d-2) n^(d+1) + 16 d n^d + n^d)."""
    return float(ncells) * (2 * (3 * d - 2) * n ** (d + 1) + 16 * d * n ** d + n ** d)


def solve_flops(d: int, m: int, n_sub: int) -> float:
    """n_sub (2d m^d (2m-1) + 3 m^d): the reference's local-solver count
    including the omega scale and add (`fastdiag.py:503-507`, `625-628`)."""
    return float(n_sub) * (2 * d * m ** d * (2 * m - 1) + 3 * m ** d)


def step_work(kind: str, d: int, k: int, dims: tuple[int, ...]) -> tuple[float, float]:
    """(flops, compulsory HBM bytes) of one smoothing step."""
    n = k + 1
    ncells = 1
    for v in dims:
        ncells *= v
    ndofs = ncells * n ** d
    fres = residual_flops_min(d, n, ncells)
    if kind in ("acs", "mcs"):
        fsolve = solve_flops(d, n, ncells)
        kappa = 1.0
    else:
        npatch = 1
        for v in dims:
            npatch *= max(0, v - 1)
        fsolve = solve_flops(d, 2 * n, npatch)
        kappa = 1.0
        if kind == "mvs":
            kappa = float(2 ** d)
            for v in dims:
                kappa *= (v - 1) / v
    return kappa * fres + fsolve, kappa * 24.0 * ndofs


def _contraction(m: int, eo: bool) -> float:
    """flops of one length-m fiber contraction: dense m(2m-1); even/odd split
    m^2 (two (m/2)^2 FMA blocks) + m (sums/differences or recombination)."""
    return float(m * m + m) if eo else float(m * (2 * m - 1))


def executed_step_flops(kind: str, d: int, k: int, dims: tuple[int, ...],
                        eo_fdm: bool, eo_res: bool) -> float:
    """Flops the device kernels execute for one step, counting the even/odd
    split of interior-digit contractions (tables.device_tables) as used."""
    n = k + 1
    ncells = 1
    for v in dims:
        ncells *= v
    fib = n ** (d - 1)
    # residual per cell: d stiffness + (2d-1) mass contractions (3D: 3 + 5),
    # rank-2 face couplings and the subtraction (SURVEY 8(d) convention)
    nmass = 5 if d == 3 else 2
    res = 0.0
    for t in range(d):
        inter = max(0, dims[t] - 2) / dims[t]
        res += fib * (inter * _contraction(n, eo_res and n % 2 == 0)
                      + (1 - inter) * _contraction(n, False)) * ncells
    res += nmass * fib * _contraction(n, eo_res and n % 2 == 0) * ncells
    res += ncells * (16 * d * n ** d + n ** d)
    if kind in ("acs", "mcs"):
        m, nsub, fr = n, ncells, [max(0, v - 2) / v for v in dims]
        eo_ok = eo_fdm and n % 2 == 0
    else:
        m = 2 * n
        nsub = 1
        for v in dims:
            nsub *= max(0, v - 1)
        fr = [max(0, v - 3) / max(1, v - 1) for v in dims]
        eo_ok = eo_fdm
    mf = m ** (d - 1)
    sol = 0.0
    for t in range(d):
        per = fr[t] * _contraction(m, eo_ok) + (1 - fr[t]) * _contraction(m, False)
        sol += 2 * mf * per
    sol = nsub * (sol + 3 * m ** d)
    kappa = 1.0
    if kind == "mvs":
        kappa = float(2 ** d)
        for v in dims:
            kappa *= (v - 1) / v
    return kappa * res + sol
