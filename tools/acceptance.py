"""Reproduce the reference's Cartesian iteration-count runs (acceptance
criteria 3-5, `test_acceptance.py:111-181`) on the device and print one JSON
line per level: smoother, dims, dofs, iterations, fractional count, wall time.

    python tools/acceptance.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1910_11239_b200.experiment import ExperimentConfig, run_experiment  # noqa: E402

TARGETS = {"acs_2d_k3": 14.5, "mcs_2d_k3": 7.3, "mvs_2d_k3": 2.5, "acs_2d_k7": 18.7,
           "mcs_2d_k7": 9.7, "mvs_2d_k7": 2.1, "acs_3d_k3": 17.1, "mcs_3d_k3": 8.6,
           "mvs_3d_k3": 2.4}
RUNS = (("acs_2d_k3", 2, 3, 6, 8), ("mcs_2d_k3", 2, 3, 6, 8), ("mvs_2d_k3", 2, 3, 6, 8),
        ("acs_2d_k7", 2, 7, 7, 7), ("mcs_2d_k7", 2, 7, 7, 7), ("mvs_2d_k7", 2, 7, 7, 7),
        ("acs_3d_k3", 3, 3, 3, 3), ("mcs_3d_k3", 3, 3, 3, 3), ("mvs_3d_k3", 3, 3, 3, 3),
        ("avs_2d_k3", 2, 3, 6, 8), ("avs_3d_k3", 3, 3, 3, 4), ("mvs_3d_k5", 3, 5, 3, 4))
for key, d, k, l0, l1 in RUNS:
    sm = key.split("_")[0]
    # additive vertex patches need two smoothing steps per V-cycle level to be
    # a convergent preconditioner (the reference's test_multigrid.py:175-190)
    m = 2 if sm == "avs" else 1
    # and omega <= 2^-d (test_multigrid.py:178-180): the reference's default
    # 0.25 (bench.py:93-102) is 2^-d in 2D only; at 0.25 the 3D AVS
    # preconditioned CG does not converge in 200 iterations
    om = 2.0 ** -d if sm == "avs" else None
    for r in run_experiment(ExperimentConfig(dim=d, degree=k, level_min=l0, level_max=l1,
                                             smoother=sm, omega=om, m_pre=m, m_post=m)):
        print(json.dumps({"run": key, "level": r.level, "cells_per_dim": 2 * 2 ** r.level,
                          "dofs": r.dofs, "solver": r.config["solver"], "omega": r.config["omega"],
                          "iterations": r.iterations, "nu_frac": round(r.nu_frac, 3),
                          "reference_target": TARGETS.get(key), "converged": r.converged,
                          "wall_s": round(r.wall_time, 3)}), flush=True)

# criterion 6: distorted meshes (test_acceptance.py:187-220)
for key, lv0, lv1, sm, om, m, target in (("dist_acs1_2d_k3", 3, 5, "acs", 0.5, 1, {3: 38.7, 4: 37.6, 5: 37.6}),
                                         ("dist_mcs1_2d_k3", 4, 4, "mcs", 0.75, 1, {4: 23.5}),
                                         ("dist_acs2_2d_k3", 3, 3, "acs", 0.5, 2, {})):
    for r in run_experiment(ExperimentConfig(dim=2, degree=3, level_min=lv0, level_max=lv1,
                                             smoother=sm, mesh_kind="distorted", omega=om,
                                             m_pre=m, m_post=m, max_it=120)):
        print(json.dumps({"run": key, "level": r.level, "coarse_cells": 32,
                          "cells_per_dim": 32 * 2 ** r.level, "dofs": r.dofs,
                          "solver": r.config["solver"], "iterations": r.iterations,
                          "nu_frac": round(r.nu_frac, 3),
                          "reference_target": target.get(r.level), "converged": r.converged,
                          "wall_s": round(r.wall_time, 3)}), flush=True)
