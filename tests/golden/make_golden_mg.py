"""Generate the multigrid / Krylov golden fixtures from the reference itself
(the V-cycle and CG around the smoothing step).

Run in the build container (the reference exists only there):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_mg.py

Imports the unmodified reference (`dgmg.multigrid`, `dgmg.krylov`) and
records, for seeded inputs (`default_rng(seed).uniform(-1, 1)`, regenerated
by the tests, not stored):

- the 1D embeddings E^0, E^1 (`multigrid.py:51-55`) for k = 1..7, 15;
- prolongation / restriction outputs (`multigrid.py:91-130`);
- direct coarse solves (`multigrid.py:148-293`), and the Chebyshev-CG one;
- V-cycle applications (`multigrid.py:326-350`) for all four smoother kinds;
- V-cycle-preconditioned CG residual histories and fractional iteration
  counts (`krylov.py:69-123`), the quantity of acceptance criteria 3-5;
- load vectors `compute_rhs(ctx, f, g)` (`dgop.py:800-871`) for the source
  and Dirichlet data RHS_F / RHS_G below (tests/_common.py repeats them);
- `bench.run_experiment` records (iterations, fractional iteration count,
  residual reduction) of the manufactured-problem solves at small levels.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_mg.npz")

# (name, dim, coarse cells/dir, k)  coarse level -> one refinement
TRANSFERS = [("tr_1d_q3_n3", 1, 3, 3), ("tr_2d_q3_n2", 2, 2, 3), ("tr_2d_q7_n3", 2, 3, 7),
             ("tr_3d_q2_n2", 3, 2, 2), ("tr_3d_q5_n3", 3, 3, 5), ("tr_3d_q1_n4", 3, 4, 1),
             ("tr_3d_q15_n1", 3, 1, 15), ("tr_2d_q15_n2", 2, 2, 15)]
# (name, dim, coarse, levels, k, kind, omega, m, symmetrize)
VCYCLES = [("vc_acs_2d_q3", 2, 2, 2, 3, "acs", 0.7, 1, False),
           ("vc_mcs_2d_q3", 2, 2, 2, 3, "mcs", 1.0, 1, False),
           ("vc_avs_2d_q3", 2, 2, 2, 3, "avs", 0.25, 2, False),
           ("vc_mvs_2d_q3", 2, 2, 2, 3, "mvs", 1.0, 1, True),
           ("vc_mvs_3d_q2", 3, 2, 1, 2, "mvs", 1.0, 1, False),
           ("vc_avs_3d_q3", 3, 2, 1, 3, "avs", 0.25, 1, False)]
# (name, dim, coarse, levels, k, kind, omega)
PCGS = [("cg_acs_2d_q3_L3", 2, 2, 3, 3, "acs", 0.7),
        ("cg_mcs_2d_q3_L3", 2, 2, 3, 3, "mcs", 1.0),
        ("cg_mvs_2d_q3_L3", 2, 2, 3, 3, "mvs", 1.0),
        ("cg_mvs_3d_q3_L1", 3, 2, 1, 3, "mvs", 1.0)]


def RHS_F(x):
    return np.sin(np.pi * x[:, 0]) * np.cos(0.5 * np.pi * x[:, -1]) + 0.25 * x.sum(axis=1)


def RHS_G(x):
    return x[:, 0] ** 2 - 0.5 * x[:, -1] + 0.125


# (name, dim, ncells_dim, k)
RHS = [("rhs_2d_q3_n4", 2, 4, 3), ("rhs_3d_q2_n3", 3, 3, 2), ("rhs_3d_q5_n2", 3, 2, 5),
       ("rhs_1d_q4_n5", 1, 5, 4)]


# (name, dim, k, level_min, level_max, smoother)
EXPERIMENTS = [("ex_acs_2d_k3", 2, 3, 3, 4, "acs"), ("ex_mcs_2d_k3", 2, 3, 3, 4, "mcs"),
               ("ex_mvs_2d_k3", 2, 3, 3, 4, "mvs"), ("ex_avs_2d_k3", 2, 3, 3, 3, "avs"),
               ("ex_mvs_3d_k2", 3, 2, 1, 2, "mvs"), ("ex_acs_3d_k3", 3, 3, 1, 1, "acs")]


def main() -> None:
    sys.path.insert(0, REF)
    from dgmg import dgop, krylov, mesh
    from dgmg import multigrid as mg
    from dgmg.polybasis import Basis1D
    from dgmg.smoothers import SmootherConfig

    def stack(d, coarse, levels, k, **kw):
        h = mesh.build_hierarchy(d, coarse, levels)
        basis = Basis1D.make(k)
        ctxs = [dgop.make_context(lvl, basis, gamma_hat=1.0) for lvl in h.levels]
        return basis, ctxs, mg.VCycle(ctxs, basis, mg.MultigridConfig(**kw))

    def u(n, seed):
        return np.random.default_rng(seed).uniform(-1.0, 1.0, n)

    out = {}
    for k in (1, 2, 3, 4, 5, 6, 7, 15):
        pair = mg.build_transfer(Basis1D.make(k))
        out[f"E_k{k}/e0"] = pair.e0
        out[f"E_k{k}/e1"] = pair.e1
    for name, d, nc, k in TRANSFERS:
        _, ctxs, cyc = stack(d, nc, 1, k)
        xc = u(ctxs[0].ndofs, 0)
        xf = u(ctxs[1].ndofs, 1)
        p = np.empty(ctxs[1].ndofs)
        cyc.transfers[0].prolongate(xc, p)
        r = np.empty(ctxs[0].ndofs)
        cyc.transfers[0].restrict(xf, r)
        out[name + "/P"] = p
        out[name + "/R"] = r
    for name, d, nc, k in (("cs_2d_q2_n4", 2, 4, 2), ("cs_3d_q3_n2", 3, 2, 3)):
        basis, ctxs, _ = stack(d, nc, 0, k)
        b = u(ctxs[0].ndofs, 0)
        x = np.empty_like(b)
        mg.CoarseSolver(ctxs[0], basis, mg.MultigridConfig(coarse="direct")).solve(b, x)
        out[name + "/direct"] = x
        x = np.empty_like(b)
        mg.CoarseSolver(ctxs[0], basis, mg.MultigridConfig(coarse="chebyshev_cg")).solve(b, x)
        out[name + "/cheb"] = x
    for name, d, nc, lv, k, kind, om, m, sym in VCYCLES:
        cfg = SmootherConfig(kind=kind, omega=om, m_pre=m, m_post=m, symmetrize=sym)
        _, ctxs, cyc = stack(d, nc, lv, k, smoother=cfg)
        b = u(ctxs[-1].ndofs, 0)
        out[name + "/x"] = cyc.apply(b, np.empty_like(b)).copy()
        out[name + "/meta"] = np.array([d, nc, lv, k, om, m, float(sym)])
    for name, d, nc, lv, k, kind, om in PCGS:
        cfg = SmootherConfig(kind=kind, omega=om)
        _, ctxs, cyc = stack(d, nc, lv, k, smoother=cfg)
        ctx = ctxs[-1]
        b = u(ctx.ndofs, 0)
        res = krylov.pcg(lambda x, o: dgop.apply_operator(ctx, x, out=o), b,
                         lambda r, o: cyc.apply(r, o), delta_red=1e-8, max_it=100)
        out[name + "/history"] = np.array(res.history)
        out[name + "/x"] = res.x
        out[name + "/nu_frac"] = np.array([res.nu_frac, res.iterations])
        out[name + "/meta"] = np.array([d, nc, lv, k, om])
    for name, d, nc, k in RHS:
        ctx = dgop.make_context(mesh.build_hierarchy(d, nc, 0).levels[0], Basis1D.make(k), 1.0)
        out[name + "/rhs"] = dgop.compute_rhs(ctx, RHS_F, RHS_G)
    from dgmg.bench import ExperimentConfig, run_experiment
    for name, d, k, l0, l1, smoother in EXPERIMENTS:
        recs = run_experiment(ExperimentConfig(dim=d, degree=k, level_min=l0, level_max=l1,
                                               smoother=smoother))
        out[name + "/records"] = np.array([[r.level, r.iterations, r.nu_frac, float(r.converged)]
                                           for r in recs])
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
