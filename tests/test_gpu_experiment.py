"""End-to-end solver runs on the device (the paper's iteration counts):
manufactured problem -> `dgop.compute_rhs` -> V-cycle-preconditioned CG /
GMRES, all on the GPU (`paper_1910_11239_b200.experiment`, mirror of
`dgmg.bench.run_experiment`, `bench.py:190-300`).

- small levels: iteration counts and fractional counts equal the
  reference's own records (tests/golden/make_golden_mg.py);
- the reference's acceptance criteria 3-5 (`test_acceptance.py:111-181`) at
  their own levels (2D Q3 levels 6-8, 2D Q7 level 7, 3D Q3 level 3): the
  fractional iteration counts within the reference's stated tolerances of its
  targets, converged everywhere, mesh-independent (spread <= 1), and the
  degree robustness of the MVS V-cycle.
"""
import pytest

from _common import golden_mg

from paper_1910_11239_b200.experiment import ExperimentConfig, run_experiment

pytestmark = pytest.mark.gpu
G = golden_mg()
EXS = sorted({k.split("/")[0] for k in G if k.startswith("ex_")})


@pytest.mark.parametrize("name", EXS)
def test_experiment_records_match_reference(name):
    _, smoother, dd, kk = name.split("_")
    d, k = int(dd[0]), int(kk[1:])
    ref = G[name + "/records"]
    l0, l1 = int(ref[0, 0]), int(ref[-1, 0])
    recs = run_experiment(ExperimentConfig(dim=d, degree=k, level_min=l0, level_max=l1,
                                           smoother=smoother))
    for r, (lv, it, nu, conv) in zip(recs, ref):
        assert r.level == int(lv) and r.converged == bool(conv)
        assert r.iterations == int(it)
        assert abs(r.nu_frac - nu) <= 1e-6


@pytest.fixture(scope="module")
def cartesian_runs():
    fam = {}
    for key, d, k, l0, l1, sm in (("acs_2d_k3", 2, 3, 6, 8, "acs"), ("mcs_2d_k3", 2, 3, 6, 8, "mcs"),
                                  ("mvs_2d_k3", 2, 3, 6, 8, "mvs"), ("acs_2d_k7", 2, 7, 7, 7, "acs"),
                                  ("mcs_2d_k7", 2, 7, 7, 7, "mcs"), ("mvs_2d_k7", 2, 7, 7, 7, "mvs"),
                                  ("acs_3d_k3", 3, 3, 3, 3, "acs"), ("mcs_3d_k3", 3, 3, 3, 3, "mcs"),
                                  ("mvs_3d_k3", 3, 3, 3, 3, "mvs")):
        fam[key] = run_experiment(ExperimentConfig(dim=d, degree=k, level_min=l0,
                                                   level_max=l1, smoother=sm))
    return fam


def test_criterion_3_cell_smoothers(cartesian_runs):
    """`test_acceptance.py:125-146`: ACS / MCS targets +- 1.5."""
    for key, level, target in (("acs_2d_k3", None, 14.5), ("mcs_2d_k3", None, 7.3),
                               ("acs_2d_k7", 7, 18.7), ("mcs_2d_k7", 7, 9.7),
                               ("acs_3d_k3", 3, 17.1), ("mcs_3d_k3", 3, 8.6)):
        recs = [r for r in cartesian_runs[key] if level is None or r.level == level]
        for r in recs:
            assert r.converged
            assert abs(r.nu_frac - target) <= 1.5, (key, r.level, r.nu_frac)


def test_criterion_4_mvs(cartesian_runs):
    """`test_acceptance.py:149-168`: MVS targets +- 0.5, degree robustness."""
    for key, level, target in (("mvs_2d_k3", 8, 2.5), ("mvs_2d_k7", 7, 2.1),
                               ("mvs_3d_k3", 3, 2.4)):
        r = [r for r in cartesian_runs[key] if r.level == level][0]
        assert r.converged and abs(r.nu_frac - target) <= 0.5, (key, r.nu_frac)
    k3 = [r for r in cartesian_runs["mvs_2d_k3"] if r.level == 7][0]
    k7 = [r for r in cartesian_runs["mvs_2d_k7"] if r.level == 7][0]
    assert k7.nu_frac <= k3.nu_frac + 1e-9


def test_criterion_5_mesh_independence(cartesian_runs):
    """`test_acceptance.py:171-181`: spread over levels 6..8 <= 1."""
    for key in ("acs_2d_k3", "mcs_2d_k3", "mvs_2d_k3"):
        vals = [r.nu_frac for r in cartesian_runs[key]]
        assert max(vals) - min(vals) <= 1.0, (key, vals)
