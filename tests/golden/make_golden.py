"""Generate the golden fixtures from the reference itself.

Run in the build container (the reference exists only there):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
records its outputs for seeded inputs (`b = default_rng(seed).uniform(-1,1)`,
`x0 = default_rng(seed+1).uniform(-1,1)`); the inputs are not
stored because numpy's PCG64 streams regenerate them exactly.  The fixtures
pin the oracle (tests/test_oracle.py) and the CUDA path (tests/test_gpu_*).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")

# (name, dim, ncells_dim, k)
OPS = [("op_2d_q3_n8", 2, 8, 3), ("op_3d_q3_n4", 3, 4, 3), ("op_3d_q5_n4", 3, 4, 5),
       ("op_3d_q7_n3", 3, 3, 7), ("op_3d_q15_n2", 3, 2, 15), ("op_2d_q1_n3", 2, 3, 1),
       ("op_3d_q2_n1", 3, 1, 2), ("op_2d_q4_n1", 2, 1, 4), ("op_3d_q1_n5", 3, 5, 1)]
# (name, kind, dim, ncells_dim, k, omega, reverse)
STEPS = [("sm_acs_2d_q3_n8", "acs", 2, 8, 3, 0.7, False),
         ("sm_avs_3d_q3_n4", "avs", 3, 4, 3, 0.25, False),
         ("sm_mvs_3d_q7_n4", "mvs", 3, 4, 7, 1.0, False),
         ("sm_acs_3d_q15_n2", "acs", 3, 2, 15, 0.7, False),
         ("sm_avs_3d_q5_n4", "avs", 3, 4, 5, 0.25, False),
         ("sm_mcs_2d_q2_n6", "mcs", 2, 6, 2, 0.9, False),
         ("sm_mcs_3d_q3_n3", "mcs", 3, 3, 3, 1.0, True),
         ("sm_avs_2d_q2_n6", "avs", 2, 6, 2, 0.2, False),
         ("sm_mvs_2d_q3_n5", "mvs", 2, 5, 3, 1.0, False),
         ("sm_mvs_3d_q2_n5", "mvs", 3, 5, 2, 1.0, True),
         ("sm_acs_2d_q3_n1", "acs", 2, 1, 3, 1.0, False),
         ("sm_avs_2d_q2_n2", "avs", 2, 2, 2, 1.0, False),
         ("sm_avs_3d_q1_n6", "avs", 3, 6, 1, 0.25, False),
         ("sm_acs_3d_q5_n4", "acs", 3, 4, 5, 0.7, False)]
MAPS = [("map_3d_q3_n4", 3, 4, 3), ("map_2d_q2_n5", 2, 5, 2), ("map_3d_q1_n5", 3, 5, 1)]
COLOURS = [("col_3d_n8", 3, 8), ("col_2d_n7", 2, 7), ("col_3d_n5", 3, 5)]


def main() -> None:
    sys.path.insert(0, REF)
    from dgmg import dgop, mesh
    from dgmg import smoothers as sm
    from dgmg import fastdiag as fd
    from dgmg.polybasis import (BOUNDARY, Basis1D, interior, univariate_cell_factors,
                                univariate_patch_factors, generalized_sym_eig)

    def inputs(n, seed=0):
        b = np.random.default_rng(seed).uniform(-1.0, 1.0, n)
        x0 = np.random.default_rng(seed + 1).uniform(-1.0, 1.0, n)
        return x0, b

    out = {}
    for name, d, nc, k in OPS:
        lvl = mesh.build_hierarchy(d, nc, 0).levels[0]
        ctx = dgop.make_context(lvl, Basis1D.make(k), 1.0)
        x0, b = inputs(ctx.ndofs)
        out[name + "/Ax"] = dgop.apply_operator(ctx, x0)
        r = np.empty(ctx.ndofs)
        out[name + "/res"] = dgop.residual(ctx, x0, b, out=r).copy()
    for name, kind, d, nc, k, om, rev in STEPS:
        lvl = mesh.build_hierarchy(d, nc, 0).levels[0]
        basis = Basis1D.make(k)
        ctx = dgop.make_context(lvl, basis, 1.0)
        s = sm.make_level_smoother(ctx, basis, sm.SmootherConfig(kind=kind, omega=om))
        x0, b = inputs(ctx.ndofs)
        x = x0.copy()
        s.smooth(x, b, reverse=rev)
        out[name + "/x"] = x
        out[name + "/meta"] = np.array([d, nc, k, om, float(rev)])
    for name, d, nc, k in MAPS:
        lvl = mesh.build_hierarchy(d, nc, 0).levels[0]
        pset = fd.PatchSolverSet(lvl, Basis1D.make(k), 1.0)
        out[name + "/gidx"] = np.stack([pset.subdomain_indices(j)
                                        for j in range(len(pset.patches))])
        out[name + "/cells"] = pset.patches.cells.copy()
    for name, d, nc in COLOURS:
        lvl = mesh.build_hierarchy(d, nc, 0).levels[0]
        cp = mesh.color_patches_structured(lvl)
        out[name + "/patch_colour"] = np.concatenate(
            [np.full(len(s), c) for c, s in enumerate(cp.sets)])
        out[name + "/patch_order"] = np.concatenate(cp.sets)
        rb = mesh.color_cells_redblack(lvl)
        out[name + "/rb_order"] = np.concatenate(rb.sets)
        out[name + "/rb_sizes"] = np.array([len(s) for s in rb.sets])
    # batched solver sets (fastdiag.py:457-496, 602-628)
    lvl = mesh.build_hierarchy(3, 4, 0).levels[0]
    basis = Basis1D.make(3)
    ctx = dgop.make_context(lvl, basis, 1.0)
    _, r = inputs(ctx.ndofs, 7)
    x = np.zeros(ctx.ndofs)
    fd.CellSolverSet(lvl, basis, 1.0).solve_scaled_into(x, r, None, 1.0)
    out["cellset_3d_q3_n4/x"] = x
    x = np.zeros(ctx.ndofs)
    fd.CellSolverSet(lvl, basis, 1.0).solve_scaled_into(x, r, np.array([0, 5, 21, 63]), 0.5)
    out["cellset_sub_3d_q3_n4/x"] = x
    x = np.zeros(ctx.ndofs)
    fd.PatchSolverSet(lvl, basis, 1.0).solve_scaled_into(x, r, None, 1.0, safe_accumulate=True)
    out["patchset_3d_q3_n4/x"] = x
    # 1D factors and local inverses per digit (polybasis.py:247-341)
    for k in (1, 2, 3, 5, 7, 15):
        basis = Basis1D.make(k)
        h = 1.0 / 8
        for digit in range(4):
            left = BOUNDARY if digit & 1 else interior()
            right = BOUNDARY if digit & 2 else interior()
            f = univariate_cell_factors(basis, h, left, right, 1.0)
            out[f"f1d_k{k}_d{digit}/cell_A"] = f.stiffness
            out[f"f1d_k{k}_d{digit}/cell_M"] = f.mass
            ep = generalized_sym_eig(f.stiffness, f.mass)
            out[f"f1d_k{k}_d{digit}/cell_lam"] = ep.values
            if k <= 7:
                p = univariate_patch_factors(basis, h, h, left, right, 1.0)
                out[f"f1d_k{k}_d{digit}/patch_A"] = p.stiffness
                out[f"f1d_k{k}_d{digit}/patch_M"] = p.mass
                out[f"f1d_k{k}_d{digit}/patch_lam"] = generalized_sym_eig(p.stiffness,
                                                                          p.mass).values
    out["basis_k5/nodes"] = Basis1D.make(5).nodes
    out["basis_k5/bg"] = Basis1D.make(5).boundary_grads
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


if __name__ == "__main__":
    main()
