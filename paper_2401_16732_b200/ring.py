"""Z_q[x]/(x^n+1) on the B200 — drop-in for privinfer/ring.py.

Same public names and semantics as the reference (ring.py:1-432); every
arithmetic operation runs in libflashhe.so kernels:
  * NttPlan.fwd/inv, ntt_forward/inverse, negacyclic_mul -> K2 (fhe_ntt_*)
  * poly_add/sub/neg, scalar_mul, pointwise             -> K3 (fhe_poly_*)
  * monomial_mul (DRot), automorphism/apply_galois      -> K3 gathers
  * WidePoly lazy accumulator                            -> fhe_wide_*
Coefficients live in `ModPoly`, which can be host-resident (numpy int64,
the reference representation), device-resident (a row of a DeviceRows
stack), or both; `.coeffs` always yields the numpy view.
"""

from __future__ import annotations

import ctypes
import struct
from contextlib import contextmanager
from enum import Enum

import numpy as np
import torch

from . import _native, device
from .device import DeviceRows
from .errors import AccumulatorBudgetError, ParameterError

# ---------------------------------------------------------------------------
# op-count instrumentation (ring.py:22-40): same keys and bump points

OP_COUNTS = {"modmul": 0, "rng_draws": 0}
_counting = False


@contextmanager
def track_ops():
    global _counting
    for k in OP_COUNTS:
        OP_COUNTS[k] = 0
    _counting = True
    try:
        yield OP_COUNTS
    finally:
        _counting = False


def _bump(key, amount):
    if _counting:
        OP_COUNTS[key] += amount


class Domain(Enum):
    COEFF = "coefficient"
    EVAL = "evaluation"


class ModPoly:
    """Length-n polynomial mod `modulus` (ring.py:48-73), host and/or device."""

    __slots__ = ("_host", "_rows", "_row", "modulus", "domain")

    def __init__(self, coeffs, modulus: int, domain: Domain = Domain.COEFF):
        self.modulus = int(modulus)
        self.domain = domain
        self._rows = None
        self._row = 0
        if isinstance(coeffs, torch.Tensor):
            self._rows = DeviceRows(coeffs.reshape(1, -1).to(torch.int64))
            self._host = None
        else:
            arr = np.asarray(coeffs)
            if arr.dtype != np.int64:
                arr = arr.astype(np.int64)
            self._host = arr

    @classmethod
    def from_rows(cls, rows: DeviceRows, i: int, modulus: int, domain: Domain) -> "ModPoly":
        obj = cls.__new__(cls)
        obj.modulus = int(modulus)
        obj.domain = domain
        obj._rows = rows
        obj._row = int(i)
        obj._host = None
        return obj

    @property
    def coeffs(self) -> np.ndarray:
        if self._host is None:
            self._host = self._rows.host()[self._row]
        return self._host

    @coeffs.setter
    def coeffs(self, value):
        arr = np.asarray(value)
        self._host = arr if arr.dtype == np.int64 else arr.astype(np.int64)
        self._rows = None
        self._row = 0

    def dev(self) -> torch.Tensor:
        """1-D device view of the coefficients (uploaded on first use)."""
        if self._rows is None:
            self._rows = DeviceRows(device.to_device(self._host).reshape(1, -1))
            self._row = 0
        return self._rows.device()[self._row]

    @property
    def on_device(self) -> bool:
        return self._rows is not None

    @property
    def n(self) -> int:
        if self._host is not None:
            return len(self._host)
        return self._rows.n

    def copy(self) -> "ModPoly":
        if self._host is not None:
            return ModPoly(self._host.copy(), self.modulus, self.domain)
        return ModPoly(self.dev().clone(), self.modulus, self.domain)

    def __eq__(self, other):
        return (
            isinstance(other, ModPoly)
            and self.modulus == other.modulus
            and self.domain == other.domain
            and np.array_equal(self.coeffs, other.coeffs)
        )

    __hash__ = None

    def __repr__(self):
        where = "device" if self._host is None else "host"
        return f"ModPoly(n={self.n}, modulus={self.modulus}, domain={self.domain.name}, {where})"


def zero_poly(n: int, modulus: int, domain: Domain = Domain.COEFF) -> ModPoly:
    return ModPoly(np.zeros(n, dtype=np.int64), modulus, domain)


# ---------------------------------------------------------------------------
# row-batch helpers (the fast path: many polys per kernel launch)


def gather_rows(polys) -> torch.Tensor:
    """Device tensor [k, n] of the polys' coefficients; zero-copy when they
    are consecutive rows of one DeviceRows stack."""
    polys = list(polys)
    first = polys[0]._rows
    if first is not None and all(p._rows is first for p in polys):
        i0 = polys[0]._row
        if all(p._row == i0 + k for k, p in enumerate(polys)):
            return first.device()[i0 : i0 + len(polys)]
    if all(p._rows is None for p in polys):
        return device.to_device(np.stack([p._host for p in polys]))
    import ctypes

    rows = [p.dev() for p in polys]
    n = rows[0].shape[-1]
    out = torch.empty((len(rows), n), dtype=torch.int64, device=rows[0].device)
    ptrs = (ctypes.c_void_p * len(rows))(*[t.contiguous().data_ptr() for t in rows])
    _native.call("fhe_gather_rows", ptrs, len(rows), n, out.data_ptr(), device.stream())
    return out


def polys_from_rows(t: torch.Tensor, modulus: int, domain: Domain) -> list[ModPoly]:
    rows = DeviceRows(t)
    return [ModPoly.from_rows(rows, i, modulus, domain) for i in range(rows.rows)]


def _bitrev_array(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    idx = np.arange(n, dtype=np.int64)
    out = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        out |= ((idx >> b) & 1) << (bits - 1 - b)
    return out


def _bitrev(x: int, bits: int) -> int:
    y = 0
    for _ in range(bits):
        y = (y << 1) | (x & 1)
        x >>= 1
    return y


def ntt_rows(t: torch.Tensor, n: int, moduli, inverse: bool = False, P: int = 1,
             out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched K2 over rows [B][L][P][n] (L = len(moduli))."""
    moduli = list(moduli)
    L = len(moduli)
    rows = t.numel() // n
    B = rows // (L * P)
    if B * L * P != rows:
        raise ValueError("row count is not a multiple of L*P")
    t = t.contiguous()
    if out is None:
        out = torch.empty_like(t)
    name = "fhe_ntt_inverse" if inverse else "fhe_ntt_forward"
    _native.call(name, device.plan_array(n, moduli), L, B, P, t.data_ptr(), out.data_ptr(), device.stream())
    return out


class NttPlan:
    """Negacyclic NTT for one (n, modulus) (ring.py:88-202).

    Forward output is bit-reversed: out[i] = f(psi^(2*bitrev(i)+1)). Tables
    come from the C ABI's host path (fhe_plan_tables_host, same root search as
    ring.py:121-127); transforms run on the device.
    """

    def __init__(self, n: int, modulus: int):
        if modulus % (2 * n) != 1:
            raise ParameterError(f"modulus {modulus} is not ≡ 1 mod {2 * n}")
        self.n = n
        self.modulus = modulus
        self.native = modulus < 2**31
        lib = _native.lib()
        psi = ctypes.c_uint64()
        _native.check(lib.fhe_find_root(n, modulus, ctypes.byref(psi)))
        self.psi = int(psi.value)
        pb = np.zeros(n, dtype=np.uint64)
        ib = np.zeros(n, dtype=np.uint64)
        ninv = ctypes.c_uint64()
        _native.check(lib.fhe_plan_tables_host(n, modulus, pb.ctypes.data, ib.ctypes.data, ctypes.byref(ninv)))
        self.psi_brv = pb.astype(np.int64)
        self.ipsi_brv = ib.astype(np.int64)
        self.n_inv = int(ninv.value)
        self.exp_at_index = 2 * _bitrev_array(n) + 1
        self.index_of_exp = np.full(2 * n, -1, dtype=np.int64)
        self.index_of_exp[self.exp_at_index] = np.arange(n)

    def fwd(self, a):
        n = self.n
        _bump("modmul", n * (n.bit_length() - 1) // 2)
        return self._run(a, inverse=False)

    def inv(self, a):
        n = self.n
        _bump("modmul", n * (n.bit_length() - 1) // 2 + n)
        return self._run(a, inverse=True)

    def _run(self, a, inverse):
        if isinstance(a, torch.Tensor):
            return ntt_rows(a.reshape(-1, self.n), self.n, [self.modulus], inverse).reshape(a.shape)
        arr = np.asarray(a, dtype=np.int64)
        t = device.to_device(arr.reshape(-1, self.n))
        return ntt_rows(t, self.n, [self.modulus], inverse).cpu().numpy().reshape(arr.shape)

    def pointwise(self, a, b):
        _bump("modmul", self.n)
        dev_in = isinstance(a, torch.Tensor)
        ta = a if dev_in else device.to_device(np.asarray(a, dtype=np.int64))
        tb = b if isinstance(b, torch.Tensor) else device.to_device(np.asarray(b, dtype=np.int64))
        out = binary_rows(_native.OP_MUL, ta.reshape(1, -1), tb.reshape(1, -1), self.n, [self.modulus])
        return out.reshape(ta.shape) if dev_in else out.cpu().numpy().reshape(np.shape(a))

    def eval_perm(self, gpow: int) -> np.ndarray:
        """Permutation realising f(x) -> f(x^gpow) on NTT values (index bookkeeping)."""
        exps = self.exp_at_index * gpow % (2 * self.n)
        return self.index_of_exp[exps]


_plans: dict[tuple[int, int], NttPlan] = {}


def get_plan(n: int, modulus: int) -> NttPlan:
    key = (n, modulus)
    if key not in _plans:
        _plans[key] = NttPlan(n, modulus)
    return _plans[key]


# ---------------------------------------------------------------------------
# row kernels


def _moduli_arr(moduli):
    return _native.u64_array(moduli)


def binary_rows(op: int, a: torch.Tensor, b: torch.Tensor, n: int, moduli, P: int = 1,
                Bb: int | None = None, Pb: int | None = None, out=None) -> torch.Tensor:
    moduli = list(moduli)
    L = len(moduli)
    rows = a.numel() // n
    B = rows // (L * P)
    a = a.contiguous()
    b = b.contiguous()
    Bb = B if Bb is None else Bb
    Pb = P if Pb is None else Pb
    if b.numel() != Bb * L * Pb * n:
        raise ValueError("operand b does not match its broadcast shape")
    if out is None:
        out = torch.empty_like(a)
    _native.call("fhe_poly_binary", op, _moduli_arr(moduli), L, B, P, n, a.data_ptr(), b.data_ptr(),
                 Bb, Pb, out.data_ptr(), device.stream())
    return out


def neg_rows(a: torch.Tensor, n: int, moduli, P: int = 1) -> torch.Tensor:
    moduli = list(moduli)
    L = len(moduli)
    a = a.contiguous()
    out = torch.empty_like(a)
    B = a.numel() // n // (L * P)
    _native.call("fhe_poly_neg", _moduli_arr(moduli), L, B, P, n, a.data_ptr(), out.data_ptr(), device.stream())
    return out


def scalar_rows(a: torch.Tensor, ks, n: int, moduli, P: int = 1) -> torch.Tensor:
    moduli = list(moduli)
    L = len(moduli)
    a = a.contiguous()
    out = torch.empty_like(a)
    B = a.numel() // n // (L * P)
    _native.call("fhe_poly_scalar_mul", _moduli_arr(moduli), L, B, P, n, a.data_ptr(),
                 _native.u64_array([k % q for k, q in zip(ks, moduli)]), out.data_ptr(), device.stream())
    return out


def monomial_rows(a: torch.Tensor, shift: int, n: int, modulus: int) -> torch.Tensor:
    a = a.contiguous()
    out = torch.empty_like(a)
    R = a.numel() // n
    _native.call("fhe_poly_monomial", _moduli_arr([modulus]), 1, R, 1, n, a.data_ptr(), int(shift),
                 out.data_ptr(), device.stream())
    return out


def galois_rows(a: torch.Tensor, gpow: int, n: int, modulus: int) -> torch.Tensor:
    a = a.contiguous()
    out = torch.empty_like(a)
    R = a.numel() // n
    _native.call("fhe_poly_automorphism", _moduli_arr([modulus]), 1, R, 1, n, a.data_ptr(),
                 int(gpow) % (2 * n), out.data_ptr(), device.stream())
    return out


def _wrap(t: torch.Tensor, modulus: int, domain: Domain) -> ModPoly:
    return ModPoly.from_rows(DeviceRows(t.reshape(1, -1)), 0, modulus, domain)


# ---------------------------------------------------------------------------
# coefficient-domain ring ops (ring.py:219-334)


def _check_pair(f: ModPoly, g: ModPoly):
    if f.modulus != g.modulus:
        raise ParameterError("modulus mismatch")
    if f.n != g.n:
        raise ParameterError("length mismatch")
    if f.domain != g.domain:
        raise ParameterError("domain mismatch")


def poly_add(f: ModPoly, g: ModPoly) -> ModPoly:
    _check_pair(f, g)
    out = binary_rows(_native.OP_ADD, f.dev(), g.dev(), f.n, [f.modulus])
    return _wrap(out, f.modulus, f.domain)


def poly_sub(f: ModPoly, g: ModPoly) -> ModPoly:
    _check_pair(f, g)
    out = binary_rows(_native.OP_SUB, f.dev(), g.dev(), f.n, [f.modulus])
    return _wrap(out, f.modulus, f.domain)


def poly_neg(f: ModPoly) -> ModPoly:
    return _wrap(neg_rows(f.dev(), f.n, [f.modulus]), f.modulus, f.domain)


def scalar_mul(f: ModPoly, k: int) -> ModPoly:
    """f·k mod modulus for arbitrary integer k (ring.py:238-243)."""
    k %= f.modulus
    _bump("modmul", f.n)
    return _wrap(scalar_rows(f.dev(), [k], f.n, [f.modulus]), f.modulus, f.domain)


def ntt_forward(f: ModPoly) -> ModPoly:
    if f.domain != Domain.COEFF:
        raise ParameterError("ntt_forward expects a coefficient-domain polynomial")
    plan = get_plan(f.n, f.modulus)
    _bump("modmul", f.n * (f.n.bit_length() - 1) // 2)
    return _wrap(ntt_rows(f.dev(), plan.n, [f.modulus]), f.modulus, Domain.EVAL)


def ntt_inverse(f: ModPoly) -> ModPoly:
    if f.domain != Domain.EVAL:
        raise ParameterError("ntt_inverse expects an evaluation-domain polynomial")
    plan = get_plan(f.n, f.modulus)
    _bump("modmul", f.n * (f.n.bit_length() - 1) // 2 + f.n)
    return _wrap(ntt_rows(f.dev(), plan.n, [f.modulus], inverse=True), f.modulus, Domain.COEFF)


def negacyclic_mul(f: ModPoly, g: ModPoly) -> ModPoly:
    """f·g mod (x^n+1, modulus) via the NTT path (ring.py:269-276)."""
    _check_pair(f, g)
    n, q = f.n, f.modulus
    get_plan(n, q)
    fa = f.dev() if f.domain == Domain.EVAL else ntt_rows(f.dev(), n, [q])
    ga = g.dev() if g.domain == Domain.EVAL else ntt_rows(g.dev(), n, [q])
    prod = binary_rows(_native.OP_MUL, fa.reshape(1, -1), ga.reshape(1, -1), n, [q])
    return _wrap(ntt_rows(prod, n, [q], inverse=True), q, Domain.COEFF)


def monomial_mul(f: ModPoly, shift: int) -> ModPoly:
    """f(x)·x^(−shift) mod x^n+1: index rotation with sign flips, no modmul
    (ring.py:279-299)."""
    return _wrap(monomial_rows(f.dev(), shift, f.n, f.modulus), f.modulus, f.domain)


def automorphism(f: ModPoly, step: int) -> ModPoly:
    """f(x^(3^step)) mod x^n+1 (ring.py:316-323)."""
    return apply_galois(f, pow(3, step, 2 * f.n))


def apply_galois(f: ModPoly, gpow: int) -> ModPoly:
    if f.domain != Domain.COEFF:
        raise ParameterError("automorphism expects a coefficient-domain polynomial")
    return _wrap(galois_rows(f.dev(), gpow, f.n, f.modulus), f.modulus, Domain.COEFF)


# ---------------------------------------------------------------------------
# lazy reduction (ring.py:337-415): two int64 limbs of 30 bits per coefficient

LIMB_BITS = 30
LIMB_MASK = (1 << LIMB_BITS) - 1
WEIGHT_BUDGET = 1 << 32


class WidePoly:
    """Unreduced accumulator of scalar·poly terms, device-resident.

    `weight` tracks Σ|scalar|; a term that could overflow the limbs is
    refused before any corruption (ring.py:366-372)."""

    __slots__ = ("lo", "hi", "modulus", "weight")

    def __init__(self, n: int, modulus: int):
        self.lo = device.zeros_i64(n)
        self.hi = device.zeros_i64(n)
        self.modulus = modulus
        self.weight = 0

    @property
    def n(self) -> int:
        return self.lo.shape[0]

    def _charge(self, amount: int):
        if self.weight + amount >= WEIGHT_BUDGET:
            raise AccumulatorBudgetError(
                f"lazy accumulation budget exceeded: |scalar| sum "
                f"{self.weight + amount} ≥ {WEIGHT_BUDGET}"
            )
        self.weight += amount

    def accumulate(self, f: ModPoly, scalar: int):
        self._charge(abs(scalar))
        _native.call("fhe_wide_accumulate", self.n, f.dev().data_ptr(), ctypes.c_int64(int(scalar)),
                     self.lo.data_ptr(), self.hi.data_ptr(), device.stream())

    def accumulate_split(self, lo, hi, scalar: int):
        """Same as accumulate, for callers that pre-split the limbs once."""
        self._charge(abs(scalar))
        tlo = lo if isinstance(lo, torch.Tensor) else device.to_device(np.asarray(lo, dtype=np.int64))
        thi = hi if isinstance(hi, torch.Tensor) else device.to_device(np.asarray(hi, dtype=np.int64))
        tlo, thi = tlo.contiguous(), thi.contiguous()  # named: temporaries could be reused before the launch
        _native.call("fhe_wide_accumulate_split", self.n, tlo.data_ptr(),
                     thi.data_ptr(), ctypes.c_int64(int(scalar)), self.lo.data_ptr(),
                     self.hi.data_ptr(), device.stream())

    def add_rotated(self, other: "WidePoly", shift: int):
        """acc += other·x^(−shift), entirely in the lazy domain."""
        self._charge(other.weight)
        _native.call("fhe_wide_add_rotated", self.n, other.lo.data_ptr(), other.hi.data_ptr(),
                     ctypes.c_int64(int(shift)), self.lo.data_ptr(), self.hi.data_ptr(), device.stream())

    def finalize(self) -> ModPoly:
        """Reduce once; equals the same sum computed with per-step reduction."""
        _bump("modmul", self.n)
        out = torch.empty_like(self.lo)
        _native.call("fhe_wide_finalize", self.n, ctypes.c_uint64(self.modulus), self.lo.data_ptr(),
                     self.hi.data_ptr(), out.data_ptr(), device.stream())
        return _wrap(out, self.modulus, Domain.COEFF)


def wide_accumulate(acc: WidePoly, f: ModPoly, scalar: int) -> WidePoly:
    acc.accumulate(f, scalar)
    return acc


def finalize(acc: WidePoly) -> ModPoly:
    return acc.finalize()


# ---------------------------------------------------------------------------
# serialization: little-endian 8-byte coefficients, length-prefixed (ring.py:422-432)


def poly_to_bytes(f: ModPoly) -> bytes:
    if f.domain != Domain.COEFF:
        raise ParameterError("only coefficient-domain polynomials are serialized")
    return struct.pack("<I", f.n) + f.coeffs.astype("<u8").tobytes()


def poly_from_bytes(data: bytes, modulus: int) -> tuple[ModPoly, int]:
    (n,) = struct.unpack_from("<I", data)
    end = 4 + 8 * n
    coeffs = np.frombuffer(data[4:end], dtype="<u8").astype(np.int64)
    return ModPoly(coeffs, modulus, Domain.COEFF), end
