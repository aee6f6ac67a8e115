"""Measure the SURVEY 8(f) rows 1-2 built around the smoothing step: the
sm_100a transfer kernels, one V-cycle, and V-cycle-preconditioned CG, at the
cfg-5 discretisation (3D Q5 SIPG, 64^3 cells on the top level).

    python tools/bench_mg.py [--nc 64] [--coarse 4] [--kind avs] [--reps 20]

Prints one JSON line per measurement:
- transfer: prolongate / prolongate+accumulate / restrict between 32^3 and
  64^3 cells; algorithmic bytes = 8 B per coarse dof + 8 B per fine dof
  (+8 B per fine dof read for accumulate), achieved GB/s against the
  measured HBM peak (MEASURED_PEAKS.json);
- vcycle: VCycle.apply on the hierarchy coarse^3 .. nc^3 (device time);
- pcg: krylov.pcg with the V-cycle to ||r|| <= 1e-8 ||b||: iterations,
  fractional count, time to solution;
- cpu_vcycle: the oracle V-cycle (oracle/sipg_oracle.py, numpy) on a small
  hierarchy (the CPU reference of the same algorithm), DoF/s.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1910_11239_b200 as dg  # noqa: E402
from paper_1910_11239_b200 import krylov  # noqa: E402
from paper_1910_11239_b200 import multigrid as mg  # noqa: E402


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0


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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nc", type=int, default=64)
    ap.add_argument("--coarse", type=int, default=4)
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--kinds", default="avs:0.25:2,mvs:1.0:1",
                    help="kind:omega:m per V-cycle measurement; CG uses the last")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    peak = hbm_peak()
    d, k = 3, a.k
    basis = dg.Basis1D.make(k)

    # ---- transfer kernels (top pair of the hierarchy)
    h = dg.build_hierarchy(d, a.nc // 2, 1)
    ctxs = [dg.make_context(lvl, basis) for lvl in h.levels]
    tr = mg.LevelTransfer(mg.build_transfer(basis), ctxs[0], ctxs[1])
    nco, nfi = ctxs[0].ndofs, ctxs[1].ndofs
    xc = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, nco)).cuda()
    xf = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, nfi)).cuda()
    yf = torch.empty_like(xf)
    yc = torch.empty_like(xc)
    for name, fn, nbytes in (
            ("prolongate", lambda: tr.prolongate(xc, yf), 8 * (nco + nfi)),
            ("prolongate_accumulate", lambda: tr.prolongate(xc, yf, accumulate=True),
             8 * nco + 16 * nfi),
            ("restrict", lambda: tr.restrict(xf, yc), 8 * (nco + nfi))):
        ms = timed(fn, a.reps)
        gbs = nbytes / (ms * 1e-3) / 1e9
        print(json.dumps({"what": "transfer", "kernel": name, "coarse_cells": [a.nc // 2] * 3,
                          "fine_dofs": nfi, "ms": ms, "algorithmic_bytes": nbytes,
                          "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak}), flush=True)
    del tr, ctxs, xc, xf, yf, yc

    # ---- one V-cycle per smoother kind, V-cycle CG with the last one
    levels = int(round(np.log2(a.nc // a.coarse)))
    h = dg.build_hierarchy(d, a.coarse, levels)
    ctxs = [dg.make_context(lvl, basis) for lvl in h.levels]
    top = ctxs[-1]
    n = top.ndofs
    b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    x = torch.empty_like(b)
    for spec in a.kinds.split(","):
        kind, om, m = spec.split(":")
        cfg = dg.SmootherConfig(kind=kind, omega=float(om), m_pre=int(m), m_post=int(m))
        t0 = time.perf_counter()
        cyc = mg.VCycle(ctxs, basis, mg.MultigridConfig(smoother=cfg))
        setup_s = time.perf_counter() - t0
        ms = timed(lambda: cyc.apply(b, x), max(3, a.reps // 2))
        print(json.dumps({"what": "vcycle", "levels": [c.layout.dims[0] for c in ctxs], "k": k,
                          "smoother": kind, "omega": float(om), "m_pre": int(m),
                          "m_post": int(m), "coarse_solver": cyc.coarse.mode, "top_dofs": n,
                          "ms": ms, "dofs_per_s": n / (ms * 1e-3), "setup_s": setup_s}),
              flush=True)

    def op(u, o):
        dg.apply_operator(top, u, out=o)

    def pc(r, o):
        cyc.apply(r, o)

    krylov.pcg(op, b, pc, delta_red=1e-8, max_it=100)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = krylov.pcg(op, b, pc, delta_red=1e-8, max_it=100)
    torch.cuda.synchronize()
    t = time.perf_counter() - t0
    rn = float(torch.linalg.vector_norm(b - dg.apply_operator(top, res.x)))
    print(json.dumps({"what": "pcg", "smoother": kind, "top_dofs": n, "converged": res.converged,
                      "iterations": res.iterations, "nu_frac": res.nu_frac,
                      "s_to_solution": t, "true_rel_residual": rn / float(torch.linalg.vector_norm(b)),
                      "dofs_per_s_per_iteration": n * res.iterations / t}), flush=True)

    # ---- CPU reference of the same V-cycle (oracle port) on a small hierarchy
    if not a.no_cpu:
        from oracle.sipg_oracle import OracleVCycle
        ocyc = OracleVCycle(d, 2, 2, k, kind, float(om), int(m), int(m))
        nb = ocyc.levels[-1].ndofs
        bb = np.random.default_rng(0).uniform(-1, 1, nb)
        ocyc.apply(bb)
        ts = []
        t_all = time.perf_counter()
        while time.perf_counter() - t_all < 15.0 and len(ts) < 5:
            t0 = time.perf_counter()
            ocyc.apply(bb)
            ts.append(time.perf_counter() - t0)
        tm = min(ts)
        print(json.dumps({"what": "cpu_vcycle", "kind": "port", "smoother": kind,
                          "levels": [2, 4, 8], "k": k,
                          "top_dofs": nb, "s": tm, "dofs_per_s": nb / tm,
                          "cores": len(os.sched_getaffinity(0))}), flush=True)


if __name__ == "__main__":
    main()
