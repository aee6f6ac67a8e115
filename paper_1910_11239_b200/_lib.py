"""ctypes binding of the C ABI in include/dgmg_b200.h.

The shared library `libdgmg_b200.so` is built in-tree by
`__graft_entry__.build()` (nvcc, sm_100a).  There is no CPU fallback: if the
library or a GPU is missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .tables import LevelTables, SingularLocalSolverError, device_tables

_HERE = os.path.dirname(os.path.abspath(__file__))
# DGB_LIB selects another build of the same ABI (e.g. the experimental
# variants, __graft_entry__.build() with DGB_EXPERIMENTAL=1)
LIB_PATH = os.environ.get("DGB_LIB") or os.path.join(_HERE, "libdgmg_b200.so")

DG_OK, DG_EINVAL, DG_ESINGULAR, DG_ECUDA, DG_EUNSUPPORTED = 0, 1, 2, 3, 4
KINDS = {"acs": 0, "mcs": 1, "avs": 2, "mvs": 3}
_PATCH_CELLS = 100  # dg_colour_list kind for "cells covered by patch colour"

EXPORTS = (
    "dg_last_error", "dg_version", "dg_level_create", "dg_level_destroy",
    "dg_level_ndofs", "dg_apply", "dg_residual", "dg_residual_cells",
    "dg_cell_fdm", "dg_patch_fdm", "dg_num_colours", "dg_colour_list",
    "dg_patch_gather_map", "dg_smooth", "dg_last_launch_count", "dg_flow_enabled",
    "dg_build_flags",
    "dg_prolongate", "dg_restrict", "dg_cg_update", "dg_xpby", "dg_dot", "dg_solve_range",
    "dg_mvs_range", "dg_dist_apply", "dg_dist_cell_fdm",
    "dg_mode_contract", "dg_canonical_tensor", "dg_kron_scale",
)


class DeviceError(RuntimeError):
    """CUDA failure reported by the extension."""


class LevelDesc(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("degree", ctypes.c_int),
                ("ncells", ctypes.c_int * 3), ("z_begin", ctypes.c_int),
                ("z_count", ctypes.c_int), ("own_begin", ctypes.c_int),
                ("own_end", ctypes.c_int), ("res_begin", ctypes.c_int),
                ("res_end", ctypes.c_int), ("pv_begin", ctypes.c_int),
                ("pv_end", ctypes.c_int)]


_dp = ctypes.POINTER(ctypes.c_double)


class Tables(ctypes.Structure):
    _fields_ = [("mass", _dp), ("adiag", _dp), ("bg", _dp),
                ("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("betap", ctypes.c_double), ("cell_z", _dp), ("cell_zt", _dp),
                ("cell_invsum", _dp), ("patch_z", _dp), ("patch_zt", _dp),
                ("patch_invsum", _dp), ("cell_eo", _dp), ("patch_eo", _dp),
                ("res_eo", _dp)]


_lib = None


def load() -> ctypes.CDLL:
    """Load (once) and type the extension; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i64, c_int, c_double = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    sig = {
        "dg_last_error": ([], ctypes.c_char_p),
        "dg_version": ([], c_int),
        "dg_level_create": ([ctypes.POINTER(LevelDesc), ctypes.POINTER(Tables),
                             ctypes.POINTER(vp)], c_int),
        "dg_level_destroy": ([vp], c_int),
        "dg_level_ndofs": ([vp], i64),
        "dg_apply": ([vp, vp, vp, c_int, c_int, vp], c_int),
        "dg_residual": ([vp, vp, vp, vp, c_int, c_int, vp], c_int),
        "dg_residual_cells": ([vp, vp, vp, vp, vp, i64, vp], c_int),
        "dg_cell_fdm": ([vp, vp, vp, c_double, vp, i64, vp], c_int),
        "dg_patch_fdm": ([vp, vp, vp, c_double, vp, i64, c_int, vp], c_int),
        "dg_num_colours": ([vp, c_int], c_int),
        "dg_colour_list": ([vp, c_int, c_int, ctypes.POINTER(vp),
                            ctypes.POINTER(i64)], c_int),
        "dg_patch_gather_map": ([vp, vp, i64, vp, vp], c_int),
        "dg_smooth": ([vp, c_int, c_double, c_int, vp, vp, vp, c_int, vp], c_int),
        "dg_last_launch_count": ([vp], i64),
        "dg_flow_enabled": ([vp], c_int),
        "dg_build_flags": ([], c_int),
        "dg_prolongate": ([c_int, c_int, ctypes.POINTER(c_int), _dp, _dp, vp, vp, c_int, vp],
                          c_int),
        "dg_restrict": ([c_int, c_int, ctypes.POINTER(c_int), _dp, _dp, vp, vp, vp], c_int),
        "dg_cg_update": ([vp, vp, vp, vp, c_double, i64, vp, vp, vp], c_int),
        "dg_xpby": ([vp, c_double, vp, i64, vp], c_int),
        "dg_dot": ([vp, vp, i64, vp, vp, vp], c_int),
        "dg_solve_range": ([vp, c_int, c_double, vp, vp, c_int, c_int, vp], c_int),
        "dg_mvs_range": ([vp, c_int, c_int, c_double, vp, vp, vp, c_int, c_int, vp], c_int),
        "dg_dist_apply": ([vp, vp, vp, vp, vp], c_int),
        "dg_dist_cell_fdm": ([c_int, c_int, i64, vp, vp, vp, vp, c_double, vp, i64, vp], c_int),
        "dg_mode_contract": ([vp, vp, vp, i64, c_int, c_int, i64, c_int, vp], c_int),
        "dg_canonical_tensor": ([c_int, c_int, ctypes.POINTER(c_int), vp, vp, c_int, vp], c_int),
        "dg_kron_scale": ([vp, vp, vp, vp, c_int, c_int, c_int, vp], c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == DG_OK:
        return
    msg = _lib.dg_last_error().decode() if _lib is not None else "extension error"
    if rc == DG_EINVAL:
        raise ValueError(msg)
    if rc == DG_ESINGULAR:
        raise SingularLocalSolverError(msg)
    if rc == DG_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise DeviceError(msg)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


class DeviceLevel:
    """Owns a `dg_level_t` (device tables + colour lists) for one window."""

    def __init__(self, tables: LevelTables, dims: tuple[int, ...],
                 z_begin: int = 0, z_count: int | None = None,
                 own: tuple[int, int] | None = None,
                 res: tuple[int, int] | None = None,
                 pv: tuple[int, int] | None = None, use_eo: bool | None = None):
        lib = load()
        if use_eo is None:
            use_eo = os.environ.get("DGB_EO", "1") != "0"
        d = tables.dim
        last = dims[-1]
        z_count = last - z_begin if z_count is None else z_count
        own = (z_begin, z_begin + z_count) if own is None else own
        res = own if res is None else res
        pv = (1, last - 1) if pv is None else pv
        desc = LevelDesc()
        desc.dim = d
        desc.degree = tables.degree
        for t in range(3):
            desc.ncells[t] = dims[t] if t < d else 1
        desc.z_begin, desc.z_count = z_begin, z_count
        desc.own_begin, desc.own_end = own
        desc.res_begin, desc.res_end = res
        desc.pv_begin, desc.pv_end = pv
        keep = []

        def arr(a):
            if a is None:
                return None
            c = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(c)
            return _ptr(c)

        dt = device_tables(tables, tuple(dims), use_eo=use_eo)
        t = Tables()
        t.mass = arr(tables.mass)
        t.adiag = arr(tables.adiag)
        t.bg = arr(tables.bg)
        t.alpha, t.beta, t.betap = tables.alpha, tables.beta, tables.betap
        t.cell_z = arr(dt.cell_z)
        t.cell_zt = arr(np.transpose(dt.cell_z, (0, 2, 1)))
        t.cell_invsum = arr(dt.cell_invsum)
        t.cell_eo = arr(dt.cell_eo)
        t.res_eo = arr(dt.res_eo)
        if dt.patch_z is not None:
            t.patch_z = arr(dt.patch_z)
            t.patch_zt = arr(np.transpose(dt.patch_z, (0, 2, 1)))
            t.patch_invsum = arr(dt.patch_invsum)
            t.patch_eo = arr(dt.patch_eo)
        self.eo = {"cell": dt.cell_eo is not None, "patch": dt.patch_eo is not None,
                   "residual": dt.res_eo is not None}
        h = ctypes.c_void_p()
        check(lib.dg_level_create(ctypes.byref(desc), ctypes.byref(t), ctypes.byref(h)))
        self._lib = lib
        self.handle = h
        self.desc = desc
        self.dims = tuple(dims)
        self.dim = d
        self.ndofs = int(lib.dg_level_ndofs(h))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.dg_level_destroy(h)
            except Exception:
                pass
            self.handle = None

    def colour_list(self, kind: str, colour: int):
        """(device pointer, count) of a colour list owned by the level."""
        ptr = ctypes.c_void_p()
        cnt = ctypes.c_int64()
        k = _PATCH_CELLS if kind == "patch_cells" else KINDS[kind]
        check(self._lib.dg_colour_list(self.handle, k, colour, ctypes.byref(ptr),
                                       ctypes.byref(cnt)))
        return ptr.value, int(cnt.value)

    def num_colours(self, kind: str) -> int:
        return int(self._lib.dg_num_colours(self.handle, KINDS[kind]))
