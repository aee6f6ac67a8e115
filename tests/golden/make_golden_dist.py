"""Golden fixtures for the distorted-mesh operator from
the reference itself (run in the build container):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_dist.py

For the reference's criterion-1 cases (`test_acceptance.py:33-59`: 2D level 2
k = 1..3, 3D level 1 k = 1, 2, distortion 0.25, seed 2024, gamma_hat 4) and
two larger ones, records the distorted vertex grids of every level and
`apply_operator` on seeded inputs (`default_rng(seed).uniform(-1, 1)`).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_dist.npz")
# (name, dim, coarse, level, k)
CASES = [("dop_2d_k1_l2", 2, 2, 2, 1), ("dop_2d_k2_l2", 2, 2, 2, 2), ("dop_2d_k3_l2", 2, 2, 2, 3),
         ("dop_3d_k1_l1", 3, 2, 1, 1), ("dop_3d_k2_l1", 3, 2, 1, 2), ("dop_3d_k3_l2", 3, 2, 2, 3),
         ("dop_2d_k4_l3", 2, 4, 3, 4)]


def main() -> None:
    sys.path.insert(0, REF)
    from dgmg import dgop, mesh
    from dgmg.polybasis import Basis1D

    out = {}
    for name, d, coarse, level, k in CASES:
        hier = mesh.distort(mesh.build_hierarchy(d, coarse, level), 0.25, rng_seed=2024)
        lvl = hier.levels[level]
        ctx = dgop.make_context(lvl, Basis1D.make(k), gamma_hat=4.0)
        u = np.random.default_rng(3).uniform(-1.0, 1.0, ctx.ndofs)
        out[name + "/grid"] = lvl.vertex_grid.copy()
        out[name + "/Au"] = dgop.apply_operator(ctx, u)
        out[name + "/meta"] = np.array([d, coarse, level, k])
    # surrogate cell solver set, smoothing steps, load vector (fastdiag.py:381-496,
    # smoothers.py:131-166, dgop.py:800-871) on the 2D k = 3 and 3D k = 2 meshes
    from dgmg import fastdiag as fd
    from dgmg.smoothers import SmootherConfig, make_level_smoother
    from dgmg.bench import ExperimentConfig, manufactured, run_experiment
    for name, d, coarse, level, k in (("dsm_2d_k3", 2, 2, 2, 3), ("dsm_3d_k2", 3, 2, 1, 2)):
        hier = mesh.distort(mesh.build_hierarchy(d, coarse, level), 0.25, rng_seed=2024)
        lvl = hier.levels[level]
        basis = Basis1D.make(k)
        ctx = dgop.make_context(lvl, basis, gamma_hat=4.0)
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
        prob = manufactured(d)
        out[name + "/rhs"] = dgop.compute_rhs(ctx, prob.f, prob.g)
        out[name + "/meta"] = np.array([d, coarse, level, k])
    for name, d, k, coarse, l0, l1, sm_kind in (("dex_acs_2d_k2", 2, 2, 4, 1, 2, "acs"),
                                                ("dex_mcs_2d_k2", 2, 2, 4, 1, 1, "mcs"),
                                                ("dex_acs_3d_k2", 3, 2, 2, 1, 1, "acs")):
        recs = run_experiment(ExperimentConfig(dim=d, degree=k, coarse_cells=coarse,
                                               level_min=l0, level_max=l1, smoother=sm_kind,
                                               mesh_kind="distorted", max_it=120))
        out[name + "/records"] = np.array([[r.level, r.iterations, r.nu_frac, float(r.converged)]
                                           for r in recs])
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays")


if __name__ == "__main__":
    main()
