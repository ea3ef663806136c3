"""ctypes front end of oracle/conv_oracle.c — TEST INFRASTRUCTURE ONLY.

Used by tests/ (parity of the stacked launch on sampled output units, the C
oracle against the reference's conv goldens) and by bench.py's CPU-baseline
legs (`cpu_baseline`, `--impl reference`). Never imported by the product.

`conv_terms` restates how privinfer's `_proposed_channel` (conv.py:326-352)
enumerates the contraction: for input channel j and tap t, the source
ciphertext and the DRot step — `_tap_steps` (conv.py:245-248) plus the
channel's tile offset `tile·(j mod c_n)` for packed layouts (conv.py:342),
or the fragment's own ciphertext `j·frags + k` for fragmented ones
(conv.py:338-340).
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "liboracle.so"
_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(LIB_PATH))
        vp, i = ctypes.c_void_p, ctypes.c_int
        L.oracle_conv.restype = i
        L.oracle_conv.argtypes = [ctypes.c_uint64, i, vp, i, vp, i, i, vp, vp, i, i, vp, i, i]
        L.oracle_conv_units.restype = i
        L.oracle_conv_units.argtypes = [ctypes.c_uint64, i, vp, i, vp, i, i, vp, vp, i, i, vp, i, vp, i]
        _lib = L
    return _lib


def tap_steps(w_p: int, f_w: int) -> np.ndarray:
    """(dy − pad)·W_p + (dx − pad), row-major over (dy, dx) (conv.py:245-248)."""
    off = np.arange(f_w) - f_w // 2
    return (off[:, None] * w_p + off[None, :]).reshape(-1)


def conv_terms(layout: dict, c_i: int, f_w: int):
    """(src[K], step[K], fstride) with K = c_i·f_w², term k = j·f_w² + t."""
    taps = f_w * f_w
    steps = tap_steps(layout["w_p"], f_w)
    j = np.repeat(np.arange(c_i), taps)
    t = np.tile(np.arange(taps), c_i)
    if layout["frags"] > 1:
        src, fstride, step = j * layout["frags"], 1, steps[t]
    else:
        src, fstride, step = j // layout["c_n"], 0, steps[t] + layout["tile"] * (j % layout["c_n"])
    return src.astype(np.int32), step.astype(np.int32), fstride


def conv(q: int, n: int, cts: np.ndarray, weights2d: np.ndarray, src, step, frags: int, fstride: int,
         threads: int = 1, units=None) -> np.ndarray:
    """All output units (units=None), the first `units` (an int), or the listed
    unit indices (a sequence) of the lazy Flash contraction; returns
    [len, 2, n] uint64-valued int64 rows."""
    cts = np.ascontiguousarray(np.asarray(cts, dtype=np.int64)).view(np.uint64)
    w = np.ascontiguousarray(np.asarray(weights2d, dtype=np.int16))
    c_o, K = w.shape
    src = np.ascontiguousarray(src, dtype=np.int32)
    step = np.ascontiguousarray(step, dtype=np.int32)
    args = (ctypes.c_uint64(int(q)), n, cts.ctypes.data, cts.shape[0], w.ctypes.data, c_o, K, src.ctypes.data,
            step.ctypes.data, frags, fstride)
    if units is None or isinstance(units, (int, np.integer)):
        total = c_o * frags if units is None else int(units)
        out = np.zeros((total, 2, n), dtype=np.uint64)
        rc = lib().oracle_conv(*args, out.ctypes.data, threads, total)
    else:
        sel = np.ascontiguousarray(units, dtype=np.int32)
        out = np.zeros((len(sel), 2, n), dtype=np.uint64)
        rc = lib().oracle_conv_units(*args, out.ctypes.data, threads, sel.ctypes.data, len(sel))
    if rc:
        raise RuntimeError(f"oracle_conv failed with status {rc}")
    return out.view(np.int64)
