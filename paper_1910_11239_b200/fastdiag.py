"""Fast-diagonalisation cell and vertex-patch solver sets (device).

Mirror of `dgmg.fastdiag` on the hot path (`pkg/src/dgmg/fastdiag.py`):

- `CellSolverSet` (`fastdiag.py:314-507`) and `PatchSolverSet`
  (`fastdiag.py:510-634`) with `partition`, `solve_partitioned`,
  `solve_scaled_into`, `local_solver`, `subdomain_indices`, `classes`;
- `LocalSolver` (`fastdiag.py:103-119`) holding the per-direction 1D
  eigenpairs and the inverse Kronecker eigenvalue sums;
- `SingularLocalSolverError` (`fastdiag.py:50-51`).

`solve_partitioned(x, r, parts, omega)` computes
x[dofs of j] += omega * Z Lambda^-1 Z^T R_j r for every selected subdomain in
one `fdm_kernel` launch.  `parts` is whatever `partition()` returned (an
opaque `Selection`), or the reference's per-class list format.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._device import Staged, stream_handle
from .basis import Basis1D
from .flops import local_solver_apply_flops, local_solver_setup_flops
from .mesh import VertexPatchSet, enumerate_vertex_patches, level_dims
from .tables import SingularLocalSolverError, cell_digits, patch_digits

__all__ = [
    "LocalSolver",
    "apply_inverse",
    "EigenPair1D",
    "SingularLocalSolverError",
    "CellSolverSet",
    "PatchSolverSet",
    "Selection",
]


@dataclass(frozen=True)
class EigenPair1D:
    """Z^T A Z = diag(values), Z^T M Z = I (`polybasis.py:305-310`)."""

    vectors: np.ndarray
    values: np.ndarray


@dataclass
class LocalSolver:
    """One subdomain class's 1D eigenpairs and 1/Lambda-sum in the reference's
    reversed layout (`fastdiag.py:103-119`)."""

    kind: str
    provenance: str
    sizes: tuple
    eigenpairs: list
    inv_sum_rev: np.ndarray
    _set: object = None        # owning solver set (device execution)
    _rep: int = -1             # representative subdomain id of the class

    @property
    def ndofs(self) -> int:
        return int(np.prod(self.sizes))

    def apply_inverse(self, r):
        return apply_inverse(self, r)


def apply_inverse(solver: LocalSolver, r):
    """x = Z diag(1/sum lam) Z^T r for one subdomain (`fastdiag.py:122-133`),
    run by the level's FDM kernel on a representative subdomain of the class:
    r is placed on that subdomain's dofs of a zero level vector, solved with
    omega = 1 into a zero x, and read back through the same index map."""
    if np.asarray(r).size != solver.ndofs:
        raise ValueError("residual size does not match subdomain")
    sset = solver._set
    if sset is None:
        raise ValueError("LocalSolver is not attached to a device solver set")
    ctx = sset.ctx
    dev = ctx.dev
    n = ctx.ndofs
    shape = np.shape(r)
    rr = np.asarray(r, dtype=np.float64).reshape(-1)
    j = solver._rep
    if sset.kind == "cell":
        nd = sset.cell_dofs
        idx = torch.arange(j * nd, (j + 1) * nd, device="cuda")
    else:
        idx = torch.from_numpy(sset.gather_map(np.array([j]))[0]).cuda()
    rv = torch.zeros(n, dtype=torch.float64, device="cuda")
    xv = torch.zeros(n, dtype=torch.float64, device="cuda")
    rv[idx] = torch.from_numpy(rr).cuda()
    ids = torch.tensor([j], dtype=torch.int32, device="cuda")
    if sset.kind == "cell":
        _lib.check(dev._lib.dg_cell_fdm(dev.handle, rv.data_ptr(), xv.data_ptr(), 1.0,
                                        ids.data_ptr(), 1, stream_handle()))
    else:
        _lib.check(dev._lib.dg_patch_fdm(dev.handle, rv.data_ptr(), xv.data_ptr(), 1.0,
                                         ids.data_ptr(), 1, 0, stream_handle()))
    out = xv[idx].cpu().numpy()
    return out.reshape(shape)


class Selection:
    """Device list of subdomain ids (None = all) produced by `partition`."""

    def __init__(self, ids: np.ndarray | None):
        self.ids = ids
        self._dev = None

    @property
    def device_ids(self) -> torch.Tensor | None:
        if self._dev is None and self.ids is not None and len(self.ids):
            self._dev = torch.from_numpy(self.ids.astype(np.int32)).cuda()
        return self._dev

    def __len__(self) -> int:
        return 0 if self.ids is None else len(self.ids)


def _digits(code: int, d: int) -> list[int]:
    return [(code // 4 ** t) % 4 for t in range(d)]


def _class_codes(pos: np.ndarray, last: np.ndarray, lo: int) -> np.ndarray:
    """code = sum_t ([pos_t == lo] + 2 [pos_t == last_t]) 4^t."""
    d = pos.shape[1]
    key = (pos == lo).astype(np.int64) + 2 * (pos == last[None, :]).astype(np.int64)
    return (key * (4 ** np.arange(d, dtype=np.int64))[None, :]).sum(axis=1)


class _SolverSetBase:
    kind = ""

    def _solver_for(self, code: int) -> LocalSolver:
        t = self.ctx.tables
        d = self.dim
        digs = _digits(code, d)
        if self.kind == "cell":
            z, lam, inv, m = t.cell_z, t.cell_lam, t.cell_invsum, t.n
        else:
            z, lam, inv, m = t.patch_z, t.patch_lam, t.patch_invsum, 2 * t.n
        pairs = [EigenPair1D(z[dg].copy(), lam[dg].copy()) for dg in digs]
        inv_rev = inv[code].reshape((m,) * d).transpose(tuple(range(d - 1, -1, -1)))
        return LocalSolver(kind="cell" if self.kind == "cell" else "vertex_patch",
                           provenance="exact", sizes=(m,) * d, eigenpairs=pairs,
                           inv_sum_rev=np.ascontiguousarray(inv_rev))

    def _build_classes(self, class_of: np.ndarray) -> None:
        self.class_of = class_of
        self.classes = []
        for code in np.unique(class_of):
            rows = np.nonzero(class_of == code)[0].astype(np.int64)
            solver = self._solver_for(int(code))
            solver._set = self
            solver._rep = int(rows[0])
            self.classes.append((rows, solver))
        if self.counter is not None:
            self.counter.add("smoother_setup", len(self.classes) * local_solver_setup_flops(
                self.dim, self.ctx.basis.degree, "cell" if self.kind == "cell" else "vertex_patch"))

    def _selection(self, ids: np.ndarray | None) -> Selection:
        if ids is None:
            return Selection(None)
        return Selection(np.asarray(ids, dtype=np.int64))

    def _to_selection(self, parts) -> Selection:
        if isinstance(parts, Selection):
            return parts
        if parts is None:
            return self._selection(None)
        # reference format: one array per congruence class
        chunks = [self._part_ids(k, np.asarray(p, dtype=np.int64))
                  for k, p in enumerate(parts) if len(p)]
        ids = np.sort(np.concatenate(chunks)) if chunks else np.empty(0, dtype=np.int64)
        return self._selection(ids)


class CellSolverSet(_SolverSetBase):
    """All cell solvers of a Cartesian level (`fastdiag.py:314-507`)."""

    kind = "cell"

    def __init__(self, level, basis, gamma_hat: float, counter=None,
                 count_per_subdomain: bool = False, ctx=None):
        from .dgop import make_context

        self.ctx = ctx if ctx is not None else make_context(level, basis, gamma_hat)
        self.level = level
        self.basis = self.ctx.basis
        self.gamma_hat = gamma_hat
        self.counter = counter
        dims = level_dims(level)
        self.dim = len(dims)
        self.n1 = self.basis.n
        self.cell_dofs = self.n1 ** self.dim
        self.shared = True
        ncells = int(np.prod(dims))
        pos = np.stack(np.unravel_index(np.arange(ncells), dims[::-1])[::-1], axis=1)
        self._build_classes(_class_codes(pos, np.array(dims) - 1, 0))

    def _part_ids(self, k: int, p: np.ndarray) -> np.ndarray:
        return p  # cell parts hold cell ids (fastdiag.py:448-455)

    def local_solver(self, cell_id: int) -> LocalSolver:
        code = int(self.class_of[cell_id])
        for rows, solver in self.classes:
            if int(self.class_of[rows[0]]) == code:
                return solver
        raise KeyError(cell_id)

    def partition(self, ids) -> Selection:
        return self._selection(ids)

    def solve_partitioned(self, x, r, parts, omega: float) -> None:
        """x[dofs of selected cells] += omega A_j^-1 r_j (`fastdiag.py:457-496`)."""
        sel = self._to_selection(parts)
        dev = self.ctx.dev
        n = self.ctx.ndofs
        sx = Staged(x, n, "x")
        sr = Staged(r, n, "r")
        if sel.ids is None:
            ptr, cnt = None, 0
        else:
            ptr, cnt = (sel.device_ids.data_ptr() if len(sel) else None), len(sel)
        if sel.ids is None or cnt > 0:
            _lib.check(dev._lib.dg_cell_fdm(dev.handle, sr.ptr, sx.ptr, float(omega), ptr,
                                            cnt, stream_handle()))
        sx.finish()
        count = self.ctx.layout.ncells if sel.ids is None else cnt
        if self.counter is not None:
            self.counter.add("local_solver", count * local_solver_apply_flops(self.dim, self.n1)
                             + 2 * count * self.cell_dofs)

    def solve_scaled_into(self, x, r, ids, omega: float, safe_accumulate: bool = False) -> None:
        self.solve_partitioned(x, r, self.partition(ids), omega)


class PatchSolverSet(_SolverSetBase):
    """All vertex-patch solvers of a Cartesian level (`fastdiag.py:510-634`)."""

    kind = "vertex_patch"

    def __init__(self, level, basis, gamma_hat: float, patches: VertexPatchSet | None = None,
                 counter=None, count_per_subdomain: bool = False, ctx=None):
        from .dgop import make_context

        if not getattr(level, "cartesian", True):
            raise ValueError("vertex-patch smoothers require Cartesian levels")
        self.ctx = ctx if ctx is not None else make_context(level, basis, gamma_hat)
        self.level = level
        self.basis = self.ctx.basis
        self.gamma_hat = gamma_hat
        self.counter = counter
        self.patches = patches if patches is not None else enumerate_vertex_patches(level)
        dims = level_dims(level)
        self.dim = len(dims)
        self.m1 = 2 * self.basis.n
        self.patch_dofs = self.m1 ** self.dim
        self.cell_dofs = self.basis.n ** self.dim
        if self.ctx.tables.patch_z is None and len(self.patches):
            raise NotImplementedError("vertex patches need at least 2 cells per direction")
        v = self.patches.vertex_indices
        self._build_classes(_class_codes(v, np.array(dims) - 1, 1) if len(v)
                            else np.zeros(0, dtype=np.int64))

    def _part_ids(self, k: int, p: np.ndarray) -> np.ndarray:
        return self.classes[k][0][p]  # patch parts hold row positions per class

    def subdomain_indices(self, j: int) -> np.ndarray:
        """Global dof indices of patch j, computed on the device with the
        kernels' own index math (`fastdiag.py:579-582`)."""
        return self.gather_map(np.array([j]))[0]

    def gather_map(self, patch_ids: np.ndarray) -> np.ndarray:
        ids = torch.from_numpy(np.asarray(patch_ids, dtype=np.int32)).cuda()
        out = torch.empty((len(patch_ids), self.patch_dofs), dtype=torch.int64, device="cuda")
        dev = self.ctx.dev
        _lib.check(dev._lib.dg_patch_gather_map(dev.handle, ids.data_ptr(), len(patch_ids),
                                                out.data_ptr(), stream_handle()))
        return out.cpu().numpy()

    def local_solver(self, j: int) -> LocalSolver:
        code = int(self.class_of[j])
        for rows, solver in self.classes:
            if len(rows) and int(self.class_of[rows[0]]) == code:
                return solver
        raise KeyError(j)

    def partition(self, rows_sel) -> Selection:
        return self._selection(rows_sel)

    def solve_partitioned(self, x, r, parts, omega: float, safe_accumulate: bool = False) -> None:
        """x[patch dofs] += omega A_j^-1 R_j r (`fastdiag.py:602-628`); the
        selected patches must be write-disjoint unless safe_accumulate."""
        sel = self._to_selection(parts)
        if sel.ids is None:
            sel = self._selection(np.arange(len(self.patches)))
        cnt = len(sel)
        dev = self.ctx.dev
        n = self.ctx.ndofs
        sx = Staged(x, n, "x")
        sr = Staged(r, n, "r")
        if cnt:
            _lib.check(dev._lib.dg_patch_fdm(dev.handle, sr.ptr, sx.ptr, float(omega),
                                             sel.device_ids.data_ptr(), cnt,
                                             1 if safe_accumulate else 0, stream_handle()))
        sx.finish()
        if self.counter is not None:
            self.counter.add("local_solver", cnt * local_solver_apply_flops(self.dim, self.m1)
                             + 2 * cnt * self.patch_dofs)

    def solve_scaled_into(self, x, r, rows_sel, omega: float,
                          safe_accumulate: bool = False) -> None:
        self.solve_partitioned(x, r, self.partition(rows_sel), omega, safe_accumulate)


# keep the digit helpers importable for tests
__all__ += ["cell_digits", "patch_digits"]
