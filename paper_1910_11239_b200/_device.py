"""Device plumbing: torch for memory and streams, nothing else.

The public API accepts numpy arrays and CPU (e.g. pinned) torch tensors
(copied host<->device around the call, so that callers written for the
reference, e.g. its V-cycle, work unchanged; additive steps pipeline those
copies against the kernels, smoothers.LevelSmoother._host_step) and torch
float64 CUDA tensors (zero-copy, ordered on the current stream).
"""

from __future__ import annotations

import os

import numpy as np
import torch


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1910_11239_b200 needs a CUDA device (no CPU fallback)")


def stream_handle() -> int:
    return torch.cuda.current_stream().cuda_stream


def is_device(a) -> bool:
    return isinstance(a, torch.Tensor) and a.is_cuda


# ---------------------------------------------------------------------------
# Page-locking of recurring host buffers.  The reference's callers (its
# V-cycle, its Krylov drivers) hold one persistent numpy vector per level and
# pass the same arrays on every call; pageable memory moves at ~10-12 GB/s
# through the driver's staging and cannot overlap with the kernels, pinned
# memory at ~55 GB/s asynchronously.  A contiguous, writeable float64 array
# seen for the second time with the same address and size is therefore
# registered in place (cudaHostRegister: its pages are locked, its contents
# and address stay what they are) and unregistered when its owner is garbage
# collected.  DGB_PIN_HOST=0 turns this off, =1 registers on first sight.
# ---------------------------------------------------------------------------
_PIN_MODE = os.environ.get("DGB_PIN_HOST", "auto")
_PIN_MIN_BYTES = 1 << 20          # small vectors are not worth a registration
_pin_seen: dict = {}              # (ptr, nbytes) -> sightings
_pin_live: dict = {}              # ptr -> nbytes of our live registrations


def _owner(arr: np.ndarray):
    """The object that owns arr's memory (end of the .base chain)."""
    o = arr
    while isinstance(o, np.ndarray) and o.base is not None:
        o = o.base
    return o


_pin_pending: list = []            # unregistrations deferred out of a stream capture


def _capturing() -> bool:
    try:
        return torch.cuda.is_current_stream_capturing()
    except Exception:
        return False


def _unregister(ptr: int) -> None:
    """Finalizer of a registered array's owner.  It can fire at any point of
    the Python code, also inside a `torch.cuda.graph` capture, where
    cudaHostUnregister would invalidate the capture: deferred then."""
    if ptr not in _pin_live:
        return
    if _capturing():
        _pin_pending.append(ptr)
        return
    _pin_live.pop(ptr, None)
    try:
        torch.cuda.cudart().cudaHostUnregister(ptr)
    except Exception:  # interpreter shutdown: the context may be gone
        pass


def _drain_pending() -> None:
    while _pin_pending and not _capturing():
        ptr = _pin_pending.pop()
        if _pin_live.pop(ptr, None) is not None:
            try:
                torch.cuda.cudart().cudaHostUnregister(ptr)
            except Exception:
                pass


def maybe_pin(arr) -> bool:
    """Register arr's memory with CUDA if the policy says so; True if it is
    (now) page-locked.  Never raises: on any failure the array stays pageable."""
    if _PIN_MODE == "0" or not isinstance(arr, np.ndarray):
        return False
    if _capturing():
        return False  # no registration calls inside a stream capture
    _drain_pending()
    if (arr.dtype != np.float64 or not arr.flags.c_contiguous or not arr.flags.writeable
            or arr.nbytes < _PIN_MIN_BYTES):
        return False
    ptr, nbytes = arr.ctypes.data, arr.nbytes
    if ptr in _pin_pending:
        return False  # a dead array's range waiting to be unregistered
    if _pin_live.get(ptr) == nbytes:
        return True
    key = (ptr, nbytes)
    _pin_seen[key] = _pin_seen.get(key, 0) + 1
    if len(_pin_seen) > 4096:
        _pin_seen.clear()
    if _PIN_MODE != "1" and _pin_seen[key] < 2:
        return False
    owner = _owner(arr)
    if not isinstance(owner, np.ndarray):
        return False  # memory of a foreign owner (mmap, bytes, another library)
    import weakref
    try:
        if torch.from_numpy(arr.reshape(-1)[:1]).is_pinned():
            return True  # already page-locked by the caller
        rc = torch.cuda.cudart().cudaHostRegister(ptr, nbytes, 0)
        if int(rc) != 0:
            return False
        _pin_live[ptr] = nbytes
        weakref.finalize(owner, _unregister, ptr)
    except Exception:
        return False
    return True


class Staged:
    """A device view of a caller vector; `finish()` writes back host arrays."""

    __slots__ = ("host", "dev")

    def __init__(self, a, ndofs: int, name: str, need_copy: bool = True,
                 staging: torch.Tensor | None = None):
        if isinstance(a, torch.Tensor) and not a.is_cuda:
            # host tensor (e.g. pinned): staged like a numpy array, written back
            if a.dtype != torch.float64 or a.numel() != ndofs:
                raise ValueError(f"{name}: expected a float64 vector of the level size")
            self.host = a
            if staging is None:
                staging = torch.empty(ndofs, dtype=torch.float64, device="cuda")
            if need_copy:
                staging.copy_(a.reshape(-1), non_blocking=False)
            self.dev = staging
            return
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64:
                raise ValueError(f"{name}: expected float64")
            if a.numel() != ndofs:
                raise ValueError(f"{name}: vector size does not match level")
            if not a.is_contiguous():
                raise ValueError(f"{name}: tensor must be contiguous")
            self.host = None
            self.dev = a.view(-1)
            return
        arr = np.asarray(a)
        if arr.size != ndofs:
            raise ValueError(f"{name}: vector size does not match level")
        self.host = arr
        maybe_pin(arr)
        if staging is None:
            staging = torch.empty(ndofs, dtype=torch.float64, device="cuda")
        if need_copy:
            src = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64).reshape(-1))
            staging.copy_(src, non_blocking=False)
        self.dev = staging

    @property
    def ptr(self) -> int:
        return self.dev.data_ptr()

    def finish(self) -> None:
        if isinstance(self.host, torch.Tensor):
            self.host.view(-1).copy_(self.dev)
            return
        if self.host is not None:
            # in place like the reference, also on non-contiguous views;
            # a read-only array raises as numpy's in-place update would
            if not self.host.flags.writeable:
                raise ValueError("assignment destination is read-only")
            if self.host.flags.c_contiguous and self.host.dtype == np.float64:
                # straight into the caller's memory (no temporary host vector)
                torch.from_numpy(self.host.reshape(-1)).copy_(self.dev)
                return
            out = self.dev.cpu().numpy()
            np.copyto(self.host, out.reshape(self.host.shape))


_NVTX = os.environ.get("DGB_NVTX", "0") != "0"


class nvtx_range:
    """NVTX range around a public call when DGB_NVTX=1 (the profilers' timeline
    then shows smoothing steps, V-cycles and Krylov solves by name); a no-op
    otherwise."""

    __slots__ = ("name",)

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        if _NVTX:
            torch.cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        if _NVTX:
            torch.cuda.nvtx.range_pop()
        return False
