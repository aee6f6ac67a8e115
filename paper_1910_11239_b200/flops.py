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
