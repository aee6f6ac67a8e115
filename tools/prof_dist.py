"""One distorted-mesh operator apply and surrogate cell solve (for ncu).

    python tools/prof_dist.py --dim 2 --n 1024 --k 3
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1910_11239_b200 as dg  # noqa: E402
from paper_1910_11239_b200 import distorted as D  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dim", type=int, default=2)
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--k", type=int, default=3)
a = ap.parse_args()
h = D.distort(dg.build_hierarchy(a.dim, a.n, 0), 0.25, 1234)
ctx = D.DistortedContext(h.levels[0], dg.Basis1D.make(a.k), 4.0)
u = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda")
v = torch.empty_like(u)
D.apply_operator(ctx, u, out=v)
D.SurrogateCellSolverSet(ctx).solve_partitioned(v, u, None, 0.5)
torch.cuda.synchronize()
print("ok")
