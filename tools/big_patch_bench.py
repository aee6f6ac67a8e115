import sys, json, numpy as np, torch
sys.path.insert(0, '.')
import paper_1910_11239_b200 as dg
def timed(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
for d, nc, k, kind, om in ((3, 16, 7, "avs", 0.25), (3, 12, 9, "avs", 0.25), (3, 8, 15, "avs", 0.25), (3, 10, 11, "mvs", 1.0), (2, 64, 11, "avs", 0.25)):
    lvl = dg.build_hierarchy(d, nc, 0).levels[0]
    basis = dg.Basis1D.make(k)
    ctx = dg.make_context(lvl, basis)
    sm = dg.make_level_smoother(ctx, basis, dg.SmootherConfig(kind=kind, omega=om))
    x = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda")
    b = torch.rand(ctx.ndofs, dtype=torch.float64, device="cuda")
    ms = timed(lambda: sm.smooth(x, b))
    kt = sm.kernel_times(reps=3)
    print(json.dumps({"d": d, "nc": nc, "k": k, "kind": kind, "ndofs": ctx.ndofs, "step_ms": ms, "GDoF/s": ctx.ndofs / ms / 1e6, **{kk: v for kk, v in kt.items() if kk.endswith("_ms")}}), flush=True)
