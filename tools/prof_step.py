"""Run a few smoothing steps of a BASELINE config (for ncu / sanitizer runs).

    python tools/prof_step.py --config 5 --steps 2 [--graph]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1910_11239_b200 as dg  # noqa: E402
from bench import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--graph", action="store_true")
ap.add_argument("--nc", type=int, default=0, help="override cells per direction")
a = ap.parse_args()
c = CONFIGS[a.config]
nc = a.nc or c["nc"]
lvl = dg.build_hierarchy(c["d"], nc, 0).levels[0]
basis = dg.Basis1D.make(c["k"])
ctx = dg.make_context(lvl, basis)
sm = dg.make_level_smoother(ctx, basis, dg.SmootherConfig(kind=c["kind"], omega=c["omega"]))
sm.use_graph = a.graph
x = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, ctx.ndofs)).cuda()
b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, ctx.ndofs)).cuda()
for _ in range(a.steps):
    sm.smooth(x, b)
torch.cuda.synchronize()
print("ok", float(x.norm()))
