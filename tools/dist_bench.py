"""Distorted-mesh path timing: host setup (distortion, geometry, surrogate
eigenbases), device operator apply and surrogate cell solve, against the
Cartesian kernels on the same size.

    python tools/dist_bench.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1910_11239_b200 as dg  # noqa: E402
from paper_1910_11239_b200 import distorted as D  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


CASES = ((2, 1024, 3), (3, 32, 3), (3, 64, 2))
if os.environ.get("DIST_CASES"):  # e.g. "2,1024,1;2,1024,2"
    CASES = tuple(tuple(int(v) for v in c.split(",")) for c in os.environ["DIST_CASES"].split(";"))
for d, n, k in CASES:
    t0 = time.perf_counter()
    h = D.distort(dg.build_hierarchy(d, n, 0), 0.25, 1234)
    t1 = time.perf_counter()
    basis = dg.Basis1D.make(k)
    ctx = D.DistortedContext(h.levels[0], basis, 4.0)
    ctx._device()
    t2 = time.perf_counter()
    sset = D.SurrogateCellSolverSet(ctx)
    t3 = time.perf_counter()
    u = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda")
    v = torch.empty_like(u)
    ms_apply = timed(lambda: D.apply_operator(ctx, u, out=v))
    ms_solve = timed(lambda: sset.solve_partitioned(v, u, None, 0.5))
    cctx = dg.make_context(dg.build_hierarchy(d, n, 0).levels[0], basis)
    ms_cart = timed(lambda: dg.apply_operator(cctx, u, out=v))
    print(json.dumps({"dim": d, "cells_per_dim": n, "k": k, "dofs": ctx.ndofs,
                      "setup_distort_s": t1 - t0, "setup_geometry_s": t2 - t1,
                      "setup_surrogate_s": t3 - t2, "apply_ms": ms_apply,
                      "cell_solve_ms": ms_solve, "cartesian_apply_ms": ms_cart}), flush=True)
