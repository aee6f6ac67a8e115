"""e2e time of LevelSmoother.smooth on pinned host vectors (cfg 5) for
several pipeline chunk sizes (DGB_PIPE_LAYERS).

    python tools/e2e_sweep.py --layers 2,4,8,16
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1910_11239_b200 as dg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", default="2,4,8,16")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--config", type=int, default=5, help="BASELINE config (additive kinds: 2, 4, 5)")
a = ap.parse_args()
from bench import CONFIGS  # noqa: E402
c = CONFIGS[a.config]
lvl = dg.build_hierarchy(c["d"], c["nc"], 0).levels[0]
basis = dg.Basis1D.make(c["k"])
ctx = dg.make_context(lvl, basis)
sm = dg.make_level_smoother(ctx, basis, dg.SmootherConfig(kind=c["kind"], omega=c["omega"]))
n = ctx.ndofs
xh = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n)).pin_memory()
bh = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).pin_memory()
for c in a.layers.split(","):
    os.environ["DGB_PIPE_LAYERS"] = c
    for _ in range(2):
        sm.smooth(xh, bh)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        sm.smooth(xh, bh)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    print(json.dumps({"layers": int(c), "ms_per_step": ms, "dofs_per_s": n / (ms * 1e-3)}),
          flush=True)
# plain copies for reference: H2D of x and b, D2H of x, no compute
xd = torch.empty(n, dtype=torch.float64, device="cuda")
bd = torch.empty_like(xd)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for what in ("h2d_xb", "d2h_x"):
    torch.cuda.synchronize()
    e0.record()
    for _ in range(a.steps):
        if what == "h2d_xb":
            xd.copy_(xh, non_blocking=True)
            bd.copy_(bh, non_blocking=True)
        else:
            xh.copy_(xd, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    nbytes = 16 * n if what == "h2d_xb" else 8 * n
    print(json.dumps({"copy": what, "ms": ms, "gbs": nbytes / (ms * 1e-3) / 1e9}), flush=True)
