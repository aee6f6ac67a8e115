"""Golden fixtures for the distorted-mesh path at the degrees beyond the
register kernels (2D k = 8..15, 3D k = 5..15), from the reference itself:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_dist_big.py

Same recipe as make_golden_dist.py (distortion 0.25, seed 2024, gamma_hat 4,
`default_rng(seed).uniform(-1, 1)` inputs): `apply_operator`, the surrogate
cell solver set and one ACS / MCS step per case
(`dgop.py:432-481, 583-759`, `fastdiag.py:381-496`, `smoothers.py:131-166`).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_dist_big.npz")
# (name, dim, coarse, level, k)
CASES = [("dbig_2d_k8_l1", 2, 2, 1, 8), ("dbig_2d_k11_l1", 2, 2, 1, 11),
         ("dbig_2d_k15_l0", 2, 2, 0, 15), ("dbig_3d_k5_l1", 3, 2, 1, 5),
         ("dbig_3d_k6_l0", 3, 2, 0, 6), ("dbig_3d_k7_l1", 3, 2, 1, 7),
         ("dbig_3d_k9_l0", 3, 2, 0, 9), ("dbig_3d_k12_l0", 3, 2, 0, 12),
         ("dbig_3d_k14_l0", 3, 2, 0, 14), ("dbig_3d_k15_l0", 3, 2, 0, 15)]


def main() -> None:
    sys.path.insert(0, REF)
    from dgmg import dgop, mesh
    from dgmg import fastdiag as fd
    from dgmg.polybasis import Basis1D
    from dgmg.smoothers import SmootherConfig, make_level_smoother

    out = {}
    for name, d, coarse, level, k in CASES:
        hier = mesh.distort(mesh.build_hierarchy(d, coarse, level), 0.25, rng_seed=2024)
        lvl = hier.levels[level]
        basis = Basis1D.make(k)
        ctx = dgop.make_context(lvl, basis, gamma_hat=4.0)
        u = np.random.default_rng(3).uniform(-1.0, 1.0, ctx.ndofs)
        out[name + "/grid"] = lvl.vertex_grid.copy()
        out[name + "/Au"] = dgop.apply_operator(ctx, u)
        out[name + "/meta"] = np.array([d, coarse, level, k])
        r = np.random.default_rng(5).uniform(-1.0, 1.0, ctx.ndofs)
        x = np.zeros(ctx.ndofs)
        fd.CellSolverSet(lvl, basis, 4.0).solve_scaled_into(x, r, None, 0.5)
        out[name + "/cellset"] = x
        b = np.random.default_rng(6).uniform(-1.0, 1.0, ctx.ndofs)
        for kind, om in (("acs", 0.5), ("mcs", 0.75)):
            sm = make_level_smoother(ctx, basis, SmootherConfig(kind=kind, omega=om))
            x = np.random.default_rng(7).uniform(-1.0, 1.0, ctx.ndofs)
            sm.smooth(x, b)
            out[name + f"/{kind}"] = x
        print(name, ctx.ndofs, flush=True)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays")


if __name__ == "__main__":
    main()
