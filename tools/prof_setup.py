"""Setup cost of a distorted level (warm: a small level is built first so
CUDA / cuSOLVER initialisation is excluded): vertex perturbation, geometry
(DistortedContext) and the surrogate eigenbases (SurrogateCellSolverSet),
with a cProfile of the last two.  2D Q3, 1024^2 cells: 0.02 / 0.17 / 0.41 s.

    python tools/prof_setup.py
"""
import cProfile, pstats, time, sys
sys.path.insert(0, ".")
import torch
import paper_1910_11239_b200 as dg
from paper_1910_11239_b200 import distorted as D
h = D.distort(dg.build_hierarchy(2, 64, 0), 0.25, 1)
D.SurrogateCellSolverSet(D.DistortedContext(h.levels[0], dg.Basis1D.make(3), 4.0)); torch.cuda.synchronize()
t0 = time.perf_counter()
h = D.distort(dg.build_hierarchy(2, 32, 5), 0.25, 2024)
t1 = time.perf_counter()
pr = cProfile.Profile(); pr.enable()
ctx = D.DistortedContext(h.levels[5], dg.Basis1D.make(3), 4.0); ctx._device(); torch.cuda.synchronize()
t2 = time.perf_counter()
s = D.SurrogateCellSolverSet(ctx); torch.cuda.synchronize()
t3 = time.perf_counter()
pr.disable()
print("distort", t1 - t0, "ctx", t2 - t1, "surrogate", t3 - t2)
pstats.Stats(pr).sort_stats("cumtime").print_stats(18)
