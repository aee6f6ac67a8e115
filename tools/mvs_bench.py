"""MVS sweep time at a 3D level (restricted residual per colour + solves),
optionally with DGB_RES_BLOCK_LIST toggled.

    python tools/mvs_bench.py --nc 64 --k 5
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1910_11239_b200 as dg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nc", type=int, default=64)
ap.add_argument("--k", type=int, default=5)
ap.add_argument("--steps", type=int, default=10)
a = ap.parse_args()
lvl = dg.build_hierarchy(3, a.nc, 0).levels[0]
basis = dg.Basis1D.make(a.k)
ctx = dg.make_context(lvl, basis)
x = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda")
b = torch.rand_like(x)
for v in ("0", "1"):
    os.environ["DGB_RES_BLOCK_LIST"] = v
    sm = dg.make_level_smoother(ctx, basis, dg.SmootherConfig(kind="mvs", omega=1.0))
    for _ in range(2):
        sm.smooth(x, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        sm.smooth(x, b)
    e1.record()
    torch.cuda.synchronize()
    kt = sm.kernel_times(reps=3)
    print(json.dumps({"block_list": v, "nc": a.nc, "k": a.k, "ms_per_sweep": e0.elapsed_time(e1) / a.steps,
                      **kt}), flush=True)
