"""Host side of the distorted-mesh path (no GPU): the vertex perturbation
and midpoint refinement reproduce the reference's grids bitwise, and the
multilinear geometry is consistent."""
import os

import numpy as np
import pytest

from paper_1910_11239_b200 import distorted as D, mesh
from paper_1910_11239_b200.basis import Basis1D

G = dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                              "golden_dist.npz")))


@pytest.mark.parametrize("name", sorted({k.split("/")[0] for k in G if k.startswith("dop_")}))
def test_distort_vertex_grids_bitwise(name):
    d, coarse, level, k = (int(v) for v in G[name + "/meta"])
    h = D.distort(mesh.build_hierarchy(d, coarse, level), 0.25, 2024)
    assert np.array_equal(h.levels[level].vertex_grid, G[name + "/grid"])


def test_geometry_consistency():
    """Undistorted grid: the metric is the Cartesian diagonal vol/h^2 w, the
    face factors are the Cartesian penalty / trace weights."""
    d, n, k = 3, 3, 2
    h = D.distort(mesh.build_hierarchy(d, n, 0), 0.0, 1)
    basis = Basis1D.make(k)
    geo = D.DistortedGeometry(h.levels[0], basis, 1.0, device="cpu")
    geo.metric, geo.detjw = geo.metric.numpy(), geo.detjw.numpy()
    geo.faces = [f.numpy() for f in geo.faces]
    hh = 1.0 / n
    w = np.asarray(basis.qwts)
    wq = np.multiply.outer(np.multiply.outer(w, w), w).ravel()
    assert np.allclose(geo.metric[:, :, 0], hh ** 3 / hh ** 2 * wq[None], rtol=1e-13)
    assert np.allclose(geo.metric[:, :, 3:], 0.0, atol=1e-15)
    assert np.allclose(geo.detjw, hh ** 3 * wq[None], rtol=1e-13)
    ge = 1.0 * k * (k + 1) * 2.0 / hh
    wf = np.multiply.outer(w, w).ravel()
    assert np.allclose(geo.faces[0][..., 0], 0.5 * ge * hh ** 2 * wf[None], rtol=1e-13)


def test_surrogate_lengths_of_boxes():
    corners = np.zeros((1, 8, 3))
    for c in range(8):
        corners[0, c] = [(c & 1) * 0.5, ((c >> 1) & 1) * 0.25, ((c >> 2) & 1) * 2.0]
    assert np.allclose(D.surrogate_lengths(corners), [[0.5, 0.25, 2.0]])


def test_patch_solvers_reject_distorted_levels():
    """`test_fastdiag.py:233-240`: vertex-patch solver sets need Cartesian
    levels (ValueError)."""
    from paper_1910_11239_b200.fastdiag import PatchSolverSet
    h = D.distort(mesh.build_hierarchy(2, 2, 1), 0.2, 1)
    with pytest.raises(ValueError):
        PatchSolverSet(h.levels[1], Basis1D.make(2), 4.0)


def test_surrogate_degenerate_edge_raises():
    """`test_mesh.py:206-209`: a zero-length cell edge is rejected."""
    corners = np.array([[0.0, 0.0], [0.0, 0.0], [0.0, 1.0], [0.0, 1.0]])
    with pytest.raises(ValueError):
        D.surrogate_lengths(corners)


def test_distortion_factor_range():
    """`mesh.py:227-284`: the perturbation factor must lie in [0, 0.5)."""
    for bad in (-0.1, 0.5):
        with pytest.raises(ValueError):
            D.distort(mesh.build_hierarchy(2, 2, 0), bad, 1)


def test_dense_assembly_size_guard():
    """`test_dgop.py:301-304`: dense assembly refuses large levels."""
    from paper_1910_11239_b200 import dgop
    ctx = dgop.make_context(mesh.build_hierarchy(2, 2, 5).levels[5], Basis1D.make(3))
    with pytest.raises(ValueError):
        dgop.assemble_dense(ctx)
