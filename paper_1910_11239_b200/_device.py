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
