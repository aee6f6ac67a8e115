"""Structured Cartesian levels, vertex patches and structured colourings.

Host-side index bookkeeping for the hot path.  All maps are closed-form and
bit-exact with the reference (`pkg/src/dgmg/mesh.py`):

- cell id  c = sum_t c_t N_t^(t-1), direction 1 fastest (`mesh.py:105-112`);
- patch j <-> interior vertex v in [1, N_t-1]^d, v_1 fastest
  (`mesh.py:297-326`); patch cell for offset s: sum_t (v_t-1+s_t) stride_t,
  local slot sum_t s_t 2^(t-1);
- structured patch colour 2*parquet(v mod 2) + ((sum_t v_t//2) mod 2), sets in
  ascending colour order, empty sets dropped (`mesh.py:360-375`);
- red-black cell colour (sum_t c_t) mod 2 (`mesh.py:350-357`).

Beyond the reference (which builds cubes only, `mesh.py:142-157`) a level may
be a box with N_t cells per direction and the uniform length h in every
direction; the multi-GPU slab decomposition uses 64 x 64 x 64P boxes.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = [
    "MeshLevel",
    "MeshHierarchy",
    "VertexPatchSet",
    "ColorPartition",
    "build_hierarchy",
    "box_level",
    "enumerate_vertex_patches",
    "color_cells_redblack",
    "color_patches_structured",
    "patch_colors",
]


class MeshLevel:
    """A uniform Cartesian level: `dims[t]` cells along direction t+1, cell
    length `h` in every direction (`lengths` mirrors the reference field)."""

    def __init__(self, dim: int, dims: tuple[int, ...], h: float, index: int = 0):
        if dim not in (1, 2, 3):
            raise ValueError("dim must be 1, 2 or 3")
        if len(dims) != dim or min(dims) < 1:
            raise ValueError("need at least one cell per direction")
        self.dim = dim
        self.index = index
        self.dims = tuple(int(v) for v in dims)
        self.h = float(h)
        self.cartesian = True
        self.lengths = np.full(dim, self.h)

    @property
    def is_cube(self) -> bool:
        return len(set(self.dims)) == 1

    @property
    def ncells_dim(self) -> int:
        if not self.is_cube:
            raise ValueError("ncells_dim is defined for cube levels only; use dims")
        return self.dims[0]

    @property
    def ncells(self) -> int:
        return int(np.prod(self.dims))

    def strides(self) -> np.ndarray:
        return np.cumprod((1,) + self.dims[:-1]).astype(np.int64)

    def cell_multi_index(self, cell_id: int) -> tuple[int, ...]:
        out = []
        for t in range(self.dim):
            out.append(cell_id % self.dims[t])
            cell_id //= self.dims[t]
        return tuple(out)


@dataclass
class MeshHierarchy:
    dim: int
    coarse_cells_per_dim: int
    levels: list

    @property
    def finest(self) -> MeshLevel:
        return self.levels[-1]

    @property
    def num_levels(self) -> int:
        return len(self.levels)


def build_hierarchy(dim: int, coarse_cells_per_dim: int, max_level: int) -> MeshHierarchy:
    """Cube hierarchy on [0,1]^d with (coarse*2^l)^d cells on level l
    (`mesh.py:142-157`)."""
    if dim not in (1, 2, 3):
        raise ValueError("dim must be 1, 2 or 3")
    if coarse_cells_per_dim < 1:
        raise ValueError("need at least one coarse cell per direction")
    if max_level < 0:
        raise ValueError("max_level must be >= 0")
    levels = []
    for lvl in range(max_level + 1):
        n = coarse_cells_per_dim * 2 ** lvl
        levels.append(MeshLevel(dim, (n,) * dim, 1.0 / n, index=lvl))
    return MeshHierarchy(dim, coarse_cells_per_dim, levels)


def box_level(dims: tuple[int, ...], h: float | None = None) -> MeshLevel:
    """Box level with dims[t] cells per direction and uniform length h
    (default 1/dims[0], i.e. the unit-cube cell size of the first direction)."""
    dims = tuple(int(v) for v in dims)
    return MeshLevel(len(dims), dims, 1.0 / dims[0] if h is None else h)


def level_dims(level) -> tuple[int, ...]:
    """Per-direction cell counts of our level or a reference MeshLevel."""
    dims = getattr(level, "dims", None)
    if dims is not None:
        return tuple(dims)
    return (int(level.ncells_dim),) * int(level.dim)


class VertexPatchSet:
    """All interior-vertex patches of a level (`mesh.py:297-326`)."""

    def __init__(self, level):
        dims = level_dims(level)
        d = len(dims)
        self.level = level
        if min(dims) < 2:
            self.vertex_indices = np.empty((0, d), dtype=np.int64)
            self.cells = np.empty((0, 2 ** d), dtype=np.int64)
            return
        axes = [np.arange(1, n, dtype=np.int64) for n in dims]
        grids = np.meshgrid(*axes[::-1], indexing="ij")
        v = np.stack([g.ravel() for g in grids[::-1]], axis=-1)
        strides = np.cumprod((1,) + dims[:-1]).astype(np.int64)
        base = ((v - 1) * strides[None, :]).sum(axis=1)
        offs = np.array([sum(((c >> t) & 1) * int(strides[t]) for t in range(d))
                         for c in range(2 ** d)], dtype=np.int64)
        self.vertex_indices = v
        self.cells = base[:, None] + offs[None, :]

    def __len__(self) -> int:
        return self.cells.shape[0]


def enumerate_vertex_patches(level) -> VertexPatchSet:
    return VertexPatchSet(level)


@dataclass
class ColorPartition:
    """Disjoint index sets covering range(n_subdomains) (`mesh.py:334-347`)."""

    n_subdomains: int
    sets: list

    @property
    def num_colors(self) -> int:
        return len(self.sets)

    def validate_cover(self) -> bool:
        seen = np.concatenate(self.sets) if self.sets else np.empty(0, dtype=int)
        return len(seen) == self.n_subdomains and len(np.unique(seen)) == self.n_subdomains


def patch_colors(vertex_indices: np.ndarray) -> np.ndarray:
    """Structured colour id per patch: parquet*2 + red-black
    (`mesh.py:360-375`)."""
    v = np.asarray(vertex_indices, dtype=np.int64)
    d = v.shape[1]
    parquet = ((v % 2) * (2 ** np.arange(d, dtype=np.int64))[None, :]).sum(axis=1)
    rb = (v // 2).sum(axis=1) % 2
    return parquet * 2 + rb


def color_patches_structured(level, patches: VertexPatchSet | None = None) -> ColorPartition:
    patches = patches if patches is not None else enumerate_vertex_patches(level)
    v = patches.vertex_indices
    if len(v) == 0:
        return ColorPartition(0, [])
    col = patch_colors(v)
    ids = np.arange(len(v), dtype=np.int64)
    d = v.shape[1]
    sets = [ids[col == c] for c in range(2 ** (d + 1))]
    return ColorPartition(len(v), [s for s in sets if len(s)])


def color_cells_redblack(level) -> ColorPartition:
    dims = level_dims(level)
    idx = np.indices(dims[::-1]).sum(axis=0).ravel() % 2
    ids = np.arange(int(np.prod(dims)), dtype=np.int64)
    sets = [ids[idx == 0], ids[idx == 1]]
    return ColorPartition(len(ids), [s for s in sets if len(s)])
