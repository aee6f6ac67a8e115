"""Time the AVS step for several launch orders (DGB_AVS_WIN windows, or the
16 colour launches with DGB_AVS_COLOURS=1) at a BASELINE config.

    python tools/avs_win.py --config 5 --wins colours,0,2,4,6,8
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
from bench import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--wins", default="colours,0,2,4,6,8")
ap.add_argument("--steps", type=int, default=30)
a = ap.parse_args()
c = CONFIGS[a.config]
lvl = dg.build_hierarchy(c["d"], c["nc"], 0).levels[0]
basis = dg.Basis1D.make(c["k"])
x0 = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, lvl.ncells * basis.n ** c["d"])).cuda()
b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, x0.numel())).cuda()
ref = None
for w in a.wins.split(","):
    os.environ["DGB_AVS_COLOURS"] = "1" if w == "colours" else "0"
    os.environ["DGB_AVS_WIN"] = w if w.isdigit() else "0"
    # "atomic": one launch over all patches (bulk fp64 reduce-add), spatial order;
    # "atomic_col": same in colour order
    os.environ["DGB_AVS_ATOMIC_MAX_MDOFS"] = "100000" if w.startswith("atomic") else "64"
    os.environ["DGB_AVS_ATOMIC_ORDER"] = "0" if w == "atomic_col" else "1"
    # "ovN": overlapped residual/solve chunks of N layers; "atomic": no overlap
    os.environ["DGB_AVS_OVERLAP"] = "1" if w.startswith("ov") else "0"
    if w.startswith("ov"):
        os.environ["DGB_AVS_CHUNK"] = w[2:]
        os.environ["DGB_AVS_ATOMIC_MAX_MDOFS"] = "100000"
    ctx = dg.make_context(lvl, basis)
    sm = dg.make_level_smoother(ctx, basis, dg.SmootherConfig(kind=c["kind"], omega=c["omega"]))
    x = x0.clone()
    sm.smooth(x, b)
    torch.cuda.synchronize()
    if ref is None:
        ref = x.clone()
    diff = float(torch.linalg.vector_norm(x - ref) / torch.linalg.vector_norm(ref))
    for _ in range(3):
        sm.smooth(x, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        sm.smooth(x, b)
    e1.record()
    torch.cuda.synchronize()
    kt = sm.kernel_times(reps=5)
    print(json.dumps({"order": w, "ms_per_step": e0.elapsed_time(e1) / a.steps,
                      "rel_vs_first": diff, "launches": sm.launches_per_step(), **kt}),
          flush=True)
    del sm, ctx
