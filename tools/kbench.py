"""Time the residual / solve / step of a BASELINE config under several
DGB_* environment variants (one process, one level per variant).

    python tools/kbench.py --config 5 --variants 'A=;B=DGB_RES3_LO=1'
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
ap.add_argument("--variants", default="base=")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
c = CONFIGS[a.config]
lvl = dg.build_hierarchy(c["d"], c["nc"], 0).levels[0]
basis = dg.Basis1D.make(c["k"])
x0 = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, lvl.ncells * (c["k"] + 1) ** c["d"])).cuda()
b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, x0.numel())).cuda()
ref = {}


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for spec in a.variants.split(";"):
    name, _, env = spec.partition("=")
    saved = {}
    for kv in filter(None, env.split(",")):
        k, v = kv.split("=")
        saved[k] = os.environ.get(k)
        os.environ[k] = v
    ctx = dg.make_context(lvl, basis)
    sm = dg.make_level_smoother(ctx, basis, dg.SmootherConfig(kind=c["kind"], omega=c["omega"]))
    r = torch.empty_like(x0)
    out = {"variant": name, "env": env}
    out["residual_ms"] = timed(lambda: dg.residual(ctx, x0, b, out=r), a.reps)
    x = x0.clone()
    out["step_ms"] = timed(lambda: sm.smooth(x, b), a.reps)
    kt = sm.kernel_times(reps=10)
    out.update({k: v for k, v in kt.items() if k.endswith("_ms")})
    # agreement with the first variant
    dg.residual(ctx, x0, b, out=r)
    x = x0.clone()
    sm.smooth(x, b)
    if not ref:
        ref["r"], ref["x"] = r.clone(), x.clone()
    else:
        out["res_rel"] = float((r - ref["r"]).norm() / ref["r"].norm())
        out["step_rel"] = float((x - x0 - ref["x"] + x0).norm() / (ref["x"] - x0).norm())
    print(json.dumps(out), flush=True)
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    del ctx, sm
