"""Device plumbing: CUDA device/stream, native plan cache, row stacks.

PyTorch is used only for device memory, streams and host<->device copies;
all arithmetic runs in libflashhe.so kernels (see _native.py).
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np
import torch

from . import _native

_plans: dict[tuple[int, int, int], ctypes.c_void_p] = {}
_plan_lock = threading.Lock()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 kernels have no CPU fallback")
    _native.lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> int:
    """cudaStream_t of torch's current stream (all kernels run on it)."""
    return torch.cuda.current_stream().cuda_stream


def native_plan(n: int, q: int) -> ctypes.c_void_p:
    """fhe_plan* for (n, q) on the current device (created once, cached)."""
    dev = require_cuda().index
    key = (dev, int(n), int(q))
    p = _plans.get(key)
    if p is None:
        with _plan_lock:
            p = _plans.get(key)
            if p is None:
                p = ctypes.c_void_p()
                _native.call("fhe_plan_create", int(n), ctypes.c_uint64(int(q)), ctypes.byref(p))
                _plans[key] = p
    return p


def plan_array(n: int, moduli) -> ctypes.Array:
    plans = [native_plan(n, q) for q in moduli]
    return (ctypes.c_void_p * len(plans))(*[p.value for p in plans])


def empty_rows(rows: int, n: int) -> torch.Tensor:
    return torch.empty((rows, n), dtype=torch.int64, device=require_cuda())


def to_device(arr: np.ndarray) -> torch.Tensor:
    """Host int64 array -> device tensor (staged through pinned memory)."""
    a = np.ascontiguousarray(arr, dtype=np.int64)
    if not a.flags.writeable:
        a = a.copy()
    t = torch.from_numpy(a)
    if a.nbytes >= 1 << 16:
        t = t.pin_memory()
        return t.to(require_cuda(), non_blocking=True)
    return t.to(require_cuda())


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class DeviceRows:
    """A device tensor of polynomial rows [R, n] plus a lazily fetched host
    mirror (one bulk device->host copy serves every row)."""

    __slots__ = ("dev", "_host")

    def __init__(self, dev: torch.Tensor):
        self.dev = dev.reshape(-1, dev.shape[-1])
        self._host = None

    def host(self) -> np.ndarray:
        if self._host is None:
            h = self.dev.cpu().numpy()
            h.flags.writeable = False
            self._host = h
        return self._host

    @property
    def rows(self) -> int:
        return self.dev.shape[0]
