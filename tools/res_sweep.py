"""Residual kernel time per degree, res2 vs res3 (DGB_RES3_HI), 3D levels
of ~16M dofs.

    python tools/res_sweep.py --ks 8,9,...,15
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
ap.add_argument("--ks", default="8,9,10,11,12,13,14,15")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
for k in [int(v) for v in a.ks.split(",")]:
    n = k + 1
    nc = max(4, int(round((16.8e6 / n ** 3) ** (1 / 3))))
    lvl = dg.build_hierarchy(3, nc, 0).levels[0]
    basis = dg.Basis1D.make(k)
    ctx = dg.make_context(lvl, basis)
    x = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda")
    b = torch.rand_like(x)
    r = torch.empty_like(x)
    out = {"k": k, "nc": nc, "dofs": ctx.ndofs}
    ref = None
    for v in ("0", "1"):
        os.environ["DGB_RES3_HI"] = v
        os.environ["DGB_RES3_LO"] = v
        for _ in range(3):
            dg.residual(ctx, x, b, out=r)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            dg.residual(ctx, x, b, out=r)
        e1.record()
        torch.cuda.synchronize()
        out["res3" if v == "1" else "res2"] = e0.elapsed_time(e1) / a.reps
        if ref is None:
            ref = r.clone()
        else:
            out["rel_diff"] = float(torch.linalg.vector_norm(r - ref) / torch.linalg.vector_norm(ref))
    print(json.dumps(out), flush=True)
