"""Golden fixtures for the sizes beyond the templated kernels, from the
reference itself (run in the build container, like make_golden.py):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_big.py

Vertex-patch smoothing steps of degree 8..15 (patch tensors of 18..32 per
direction: `fastdiag.py:510-634` handles any m) and one-dimensional levels
(`mesh.py:144`, `fastdiag.py:245,284`).  Inputs as in make_golden.py
(`b = default_rng(0).uniform(-1,1)`, `x0 = default_rng(1).uniform(-1,1)`).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_big.npz")

# (name, kind, dim, ncells_dim, k, omega, reverse)
STEPS = [("sm_avs_3d_q8_n2", "avs", 3, 2, 8, 0.25, False),
         ("sm_mvs_3d_q9_n3", "mvs", 3, 3, 9, 1.0, False),
         ("sm_avs_3d_q12_n3", "avs", 3, 3, 12, 0.25, False),
         ("sm_mvs_3d_q15_n2", "mvs", 3, 2, 15, 1.0, False),
         ("sm_avs_3d_q15_n3", "avs", 3, 3, 15, 0.25, False),
         ("sm_mvs_2d_q11_n4", "mvs", 2, 4, 11, 1.0, True),
         ("sm_avs_2d_q15_n3", "avs", 2, 3, 15, 0.25, False),
         ("sm_avs_2d_q8_n5", "avs", 2, 5, 8, 0.25, False),
         # one-dimensional levels
         ("sm_acs_1d_q3_n8", "acs", 1, 8, 3, 0.7, False),
         ("sm_mcs_1d_q5_n7", "mcs", 1, 7, 5, 1.0, True),
         ("sm_avs_1d_q4_n6", "avs", 1, 6, 4, 0.5, False),
         ("sm_mvs_1d_q7_n9", "mvs", 1, 9, 7, 1.0, False),
         ("sm_mvs_1d_q15_n4", "mvs", 1, 4, 15, 1.0, True),
         ("sm_acs_1d_q1_n1", "acs", 1, 1, 1, 1.0, False)]
OPS = [("op_1d_q3_n8", 1, 8, 3), ("op_1d_q15_n3", 1, 3, 15), ("op_1d_q1_n1", 1, 1, 1),
       ("op_1d_q6_n2", 1, 2, 6)]


def main() -> None:
    sys.path.insert(0, REF)
    from dgmg import dgop, mesh
    from dgmg import smoothers as sm
    from dgmg.polybasis import Basis1D

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
        out[name + "/res"] = dgop.residual(ctx, x0, b, out=np.empty(ctx.ndofs)).copy()
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
        print(name, ctx.ndofs, flush=True)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, len(out), "arrays")


if __name__ == "__main__":
    main()
