"""ctypes binding of libflashhe.so (include/flashhe.h) — the only path to compute.

There is deliberately no CPU fallback: if the library or a CUDA device is
missing, every compute entry point raises. Status codes are mapped to the
reference's exception types (privinfer/errors.py:1-25).
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

import os

from .errors import BY_STATUS

# FLASHHE_LIB: an alternative build of the same library (development probes only)
LIB_PATH = Path(os.environ.get("FLASHHE_LIB") or Path(__file__).resolve().parent / "libflashhe.so")

FHE_OK = 0
_ERRORS = {**BY_STATUS, 5: ValueError, 6: RuntimeError}

OP_ADD, OP_SUB, OP_MUL = 0, 1, 2
MAX_LIMBS = 8

_u64 = ctypes.c_uint64
_i64 = ctypes.c_int64
_int = ctypes.c_int
_vp = ctypes.c_void_p
_PP = ctypes.POINTER(_vp)

# name -> (restype, argtypes); mirrors include/flashhe.h exactly
SIGNATURES = {
    "fhe_last_error": (ctypes.c_char_p, []),
    "fhe_abi_version": (_int, []),
    "fhe_launch_count": (_u64, []),
    "fhe_record_event": (_int, [_vp, _vp]),
    "fhe_debug_trace": (_int, [_vp]),
    "fhe_peak_imad_wide": (_int, [_int, _int, _int, _vp, _vp]),
    "fhe_peak_butterfly": (_int, [_int, _int, _int, _u64, _vp, _vp]),
    "fhe_peak_tc_i8": (_int, [_int, _int, _int, _vp, _vp]),
    "fhe_find_root": (_int, [_int, _u64, _vp]),
    "fhe_plan_tables_host": (_int, [_int, _u64, _vp, _vp, _vp]),
    "fhe_plan_create": (_int, [_int, _u64, _PP]),
    "fhe_plan_destroy": (_int, [_vp]),
    "fhe_plan_query": (_int, [_vp, _vp, _vp, _vp]),
    "fhe_ntt_forward": (_int, [_PP, _int, _int, _int, _vp, _vp, _vp]),
    "fhe_ntt_inverse": (_int, [_PP, _int, _int, _int, _vp, _vp, _vp]),
    "fhe_ntt_forward_digits": (_int, [_PP, _int, _int, _vp, _vp, _int, _int, _vp]),
    "fhe_poly_binary": (_int, [_int, _vp, _int, _int, _int, _int, _vp, _vp, _int, _int, _vp, _vp]),
    "fhe_poly_neg": (_int, [_vp, _int, _int, _int, _int, _vp, _vp, _vp]),
    "fhe_poly_mul_shoup": (_int, [_vp, _int, _int, _int, _int, _vp, _vp, _vp, _int, _int, _vp, _vp]),
    "fhe_shoup_companions": (_int, [_vp, _int, _int, _int, _int, _vp, _vp, _vp]),
    "fhe_poly_scalar_mul": (_int, [_vp, _int, _int, _int, _int, _vp, _vp, _vp, _vp]),
    "fhe_poly_monomial": (_int, [_vp, _int, _int, _int, _int, _vp, _i64, _vp, _vp]),
    "fhe_residual_add": (_int, [_u64, _int, _int, _int, _int, _vp, _vp, _vp, _vp]),
    "fhe_poly_automorphism": (_int, [_vp, _int, _int, _int, _int, _vp, _u64, _vp, _vp]),
    "fhe_poly_add_delta": (_int, [_u64, _u64, _u64, _int, _int, _vp, _vp, _vp, _vp]),
    "fhe_encrypt_combine": (_int, [_u64, _u64, _u64, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "fhe_poly_lift_centered": (_int, [_u64, _u64, _int, _int, _vp, _vp, _vp]),
    "fhe_wide_accumulate": (_int, [_int, _vp, _i64, _vp, _vp, _vp]),
    "fhe_wide_accumulate_split": (_int, [_int, _vp, _vp, _i64, _vp, _vp, _vp]),
    "fhe_wide_add_rotated": (_int, [_int, _vp, _vp, _i64, _vp, _vp, _vp]),
    "fhe_wide_finalize": (_int, [_int, _u64, _vp, _vp, _vp, _vp]),
    "fhe_decrypt_round":(_int, [_u64, _u64, _u64, _int, _int, _vp, _vp, _vp, _vp]),
    "fhe_decrypt_round_max": (_int, [_u64, _u64, _u64, _int, _int, _vp, _vp, _vp, _vp]),
    "fhe_decrypt_fused": (_int, [_vp, _int, _int, _vp, _vp, _u64, _u64, _vp, _vp, _vp]),
    "fhe_copy_many": (_int, [_int, _vp, _vp, _vp, _vp]),
    "fhe_ntt_pmult_add": (_int, [_vp, _int, _vp, _vp, _vp, _vp, _vp]),
    "fhe_gather_rows": (_int, [_vp, _int, _int, _vp, _vp]),
    "fhe_copy_2d": (_int, [_vp, ctypes.c_size_t, _vp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_size_t, _vp]),
    "fhe_zero": (_int, [_vp, ctypes.c_size_t, _vp]),
    "fhe_conv_flash": (
        _int,
        [_u64, _int, _vp, _int, _vp, _int, _int, _vp, _vp, _int, _int, _vp, _vp, _vp, _vp],
    ),
    "fhe_conv_check_budget": (_int, [_vp, _int, _int]),
    "fhe_avg_pool": (_int, [_u64, _int, _int, _int, _int, _vp, _vp, _vp]),
    "fhe_conv_tc_stack": (_int, [_u64, _int, _vp, _int, _vp, ctypes.c_size_t, _vp, _vp]),
    "fhe_conv_stream_job": (
        _int,
        [_u64, _int, _vp, _vp, ctypes.c_size_t, _vp, ctypes.c_size_t, _vp, ctypes.c_size_t, _vp, _vp, _vp, _vp,
         _vp, _vp],
    ),
    "fhe_to_montgomery": (_int, [_vp, _int, _int, _int, _int, _vp, _vp, _vp]),
    "fhe_keyswitch_apply": (_int, [_vp, _int, _int, _int, _vp, _vp, _vp, _int, _u64, _vp, _vp]),
    "fhe_keyswitch_multi": (_int, [_vp, _int, _int, _int, _vp, _vp, _int, _int, _vp, _vp, _vp, _vp]),
    "fhe_pmac": (_int, [_u64, _int, _vp, _vp, _vp, _vp, _int, _vp, _vp]),
    "fhe_rot_pmac": (
        _int,
        [_u64, _int, _int, _vp, _vp, _vp, _int, _vp, _vp, _int, _vp, _vp, _vp, _int, _vp, _vp, _vp],
    ),
    "fhe_act_client_square": (_int, [_u64, _int, _i64, _vp, _vp, _vp]),
    "fhe_act_server_const": (_int, [_u64, _int, _i64, _vp, _vp, _vp, _vp, _vp]),
    "fhe_act_gather": (_int, [_i64, _vp, _vp, _vp, _vp]),
    "fhe_act_encrypt_rows": (_int, [_u64, _u64, _u64, _int, _int, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "fhe_ct_pmult_add": (_int, [_u64, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "fhe_act_finalize": (_int, [_u64, _u64, _u64, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "fhe_act_encrypt_gather": (_int, [_u64, _u64, _u64, _int, _int, _int, _int, _vp, _vp, _vp, _vp, _vp]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load libflashhe.so (raises if it was not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                )
            h = ctypes.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name)
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def check(rc: int) -> None:
    if rc != FHE_OK:
        msg = lib().fhe_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(msg)


_fns: dict = {}


def fn(name: str):
    """The bound ctypes function (cached: the hot path avoids getattr per call)."""
    f = _fns.get(name)
    if f is None:
        f = _fns[name] = getattr(lib(), name)
    return f


def call(name: str, *args) -> None:
    rc = fn(name)(*args)
    if rc:
        check(rc)


if os.environ.get("FLASHHE_NVTX") == "1":
    # profiling aid: every C-ABI call becomes an NVTX range named after its entry
    # point (ncu --nvtx --nvtx-include "fhe_keyswitch_multi/" selects one family);
    # off by default so the hot path pays nothing
    _plain_call = call

    def call(name: str, *args) -> None:  # noqa: F811
        from torch.cuda import nvtx

        nvtx.range_push(name)
        try:
            _plain_call(name, *args)
        finally:
            nvtx.range_pop()


class ConvTcLayer(ctypes.Structure):
    """struct fhe_conv_tc_layer (include/flashhe.h)."""

    _fields_ = [
        ("in_", _vp), ("n_in", _int), ("c_i", _int), ("frags", _int), ("fstride", _int), ("chan", _vp), ("h", _int),
        ("w", _vp), ("c_o", _int), ("taps", _int), ("pos_tile", _int), ("tap_steps", _vp),
        ("bias_delta", _vp), ("bias_mask", _vp), ("out", _vp), ("rep", _int), ("tsplit", _int),
    ]


def u64_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (_u64 * len(vals))(*vals)


def launch_count() -> int:
    return int(lib().fhe_launch_count())
