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


def zeros_i64(shape) -> torch.Tensor:
    """Zeroed int64 device tensor via cudaMemsetAsync (fhe_zero), not a torch fill kernel."""
    t = torch.empty(shape, dtype=torch.int64, device=require_cuda())
    _native.call("fhe_zero", t.data_ptr(), t.numel() * 8, stream())
    return t


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


def to_device_i32(arr: np.ndarray) -> torch.Tensor:
    """Host index array -> device int32 tensor (kernel index maps)."""
    a = np.asarray(arr)
    if a.size and (a.min() < -(1 << 31) or a.max() >= 1 << 31):
        raise ValueError("index does not fit int32")
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(require_cuda())


_scratch: dict[tuple[int, str], torch.Tensor] = {}


def scratch(name: str, nbytes: int) -> int:
    """Device pointer to a named per-device scratch buffer of >= nbytes.
    Reuse is stream-ordered (every kernel runs on torch's current stream).
    Growth replaces the buffer: pointers returned earlier (and CUDA graphs
    that captured them) are then invalid. Callers size the buffer for their
    largest use before they take pointers or capture, and growth is refused
    during capture."""
    key = (torch.cuda.current_device(), name)
    t = _scratch.get(key)
    if t is None or t.numel() < nbytes:
        if t is not None:
            if torch.cuda.is_current_stream_capturing():
                raise RuntimeError(f"scratch buffer {name!r} must grow during graph capture: run once eagerly first")
            torch.cuda.synchronize()  # the old buffer may still be in use on any stream
        t = _scratch[key] = torch.empty(int(nbytes), dtype=torch.uint8, device=require_cuda())
    return t.data_ptr()


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class DeviceRows:
    """A stack of polynomial rows [R, n] living on the device, on the host, or
    both. Whichever side is missing is filled by ONE bulk copy through pinned
    host memory, so a whole ciphertext batch crosses PCIe as a single DMA in
    either direction."""

    __slots__ = ("_dev", "_host", "_pinned")

    def __init__(self, dev: torch.Tensor | None = None, host: np.ndarray | None = None, pinned=None):
        self._dev = None if dev is None else dev.reshape(-1, dev.shape[-1])
        self._host = host
        self._pinned = pinned

    @classmethod
    def from_host(cls, arr: np.ndarray, pin: bool = True) -> "DeviceRows":
        """Host-first stack; with `pin`, the rows are copied once into
        page-locked memory so the later upload is a single async DMA."""
        arr = np.asarray(arr, dtype=np.int64)
        arr = arr.reshape(-1, arr.shape[-1])
        if not pin:
            return cls(host=arr)
        t = torch.empty(arr.shape, dtype=torch.int64, pin_memory=True)
        h = t.numpy()
        h[...] = arr
        return cls(host=h, pinned=t)

    def device(self) -> torch.Tensor:
        if self._dev is None:
            src = self._pinned if self._pinned is not None else torch.from_numpy(
                np.ascontiguousarray(self._host) if self._host.flags.writeable else self._host.copy())
            self._dev = src.to(require_cuda(), non_blocking=self._pinned is not None)
        return self._dev

    dev = property(device)

    def host(self) -> np.ndarray:
        if self._host is None:
            t = torch.empty(self._dev.shape, dtype=torch.int64, pin_memory=True)
            t.copy_(self._dev, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            h = t.numpy()
            h.flags.writeable = False
            self._host, self._pinned = h, t
        return self._host

    def upload_on(self, stream: torch.cuda.Stream) -> tuple[torch.Tensor, torch.cuda.Event | None]:
        """Device rows, uploading on `stream` if they are host-only: returns
        (tensor, event the consumer must wait on; None if already resident).
        The tensor is allocated on `stream`; callers using it on another
        stream keep it alive until that stream is done (record_stream)."""
        if self._dev is not None:
            return self._dev, None
        if self._pinned is None:  # pageable host rows: stage once through pinned memory
            t = torch.empty(self._host.shape, dtype=torch.int64, pin_memory=True)
            t.numpy()[...] = self._host
            self._pinned = t
        with torch.cuda.stream(stream):
            self._dev = self._pinned.to(require_cuda(), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
        return self._dev, ev

    @classmethod
    def download_on(cls, dev: torch.Tensor, stream: torch.cuda.Stream, into: torch.Tensor | None = None) -> "DeviceRows":
        """Rows whose host copy is filled by a pinned D2H enqueued on `stream`
        (the caller orders `stream` after the producer and synchronizes it
        before reading the host side). `into`: a pinned host slice of the
        same size to fill (callers batching several downloads into one
        pinned allocation)."""
        dev = dev.reshape(-1, dev.shape[-1])
        t = torch.empty(dev.shape, dtype=torch.int64, pin_memory=True) if into is None else into.view(dev.shape)
        with torch.cuda.stream(stream):
            t.copy_(dev, non_blocking=True)
        dev.record_stream(stream)
        h = t.numpy()
        h.flags.writeable = False
        return cls(dev=dev, host=h, pinned=t)

    @property
    def rows(self) -> int:
        return (self._dev if self._dev is not None else self._host).shape[0]

    @property
    def n(self) -> int:
        return int((self._dev if self._dev is not None else self._host).shape[-1])
