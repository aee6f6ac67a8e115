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
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT}: {len(out)} arrays")


if __name__ == "__main__":
    main()
