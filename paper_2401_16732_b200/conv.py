"""Homomorphic convolution engines on the B200 — drop-in for privinfer/conv.py.

The proposed (Flash) engine, avg_pool and fully_connected all reduce to one
device primitive, K1 (`fhe_conv_flash`): an exact integer contraction of
weights against negacyclically shifted input rows, reduced once per output
coefficient. `ConvPlan` holds the per-layer device operands (int16 weights,
per-term source ciphertext and DRot step) so repeated calls are one launch.

Tile bookkeeping (TileLayout, packing, channel positions) is host-side and
follows conv.py:63-238; the conventional HRot+PMult baseline (conv.py:427-597)
runs on the hoisted key-switch kernels.
"""

from __future__ import annotations

import ctypes
import os as _os
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import _native, bfv, device, ring
from .bfv import Ciphertext, Encoding
from .errors import AccumulatorBudgetError, EncodingError, ParameterError
from .params import RingParams
from .ring import Domain

MAX_WEIGHT_BITS = 8  # |weight| < 2^8 (conv.py:28)
CONV_DECOMP_LOG = 4  # baseline switching-key digit width (conv.py:35)


@dataclass
class ConvLayerSpec:
    height: int
    width: int
    f_w: int
    c_i: int
    c_o: int
    weights: np.ndarray  # (c_o, c_i, f_w, f_w) signed ints
    weight_scale: int = 0
    bias: np.ndarray | None = None

    def __post_init__(self):
        taps = self.f_w * self.f_w
        self.weights = np.asarray(self.weights, dtype=np.int64).reshape(self.c_o, self.c_i, taps)
        if self.f_w % 2 == 0:
            raise ParameterError("kernel width must be odd")
        if self.weights.size and int(np.abs(self.weights).max()) >= 1 << MAX_WEIGHT_BITS:
            raise ParameterError(f"weights must stay below {MAX_WEIGHT_BITS} bits for lazy reduction")
        if self.bias is not None:
            self.bias = np.asarray(self.bias, dtype=np.int64)


@dataclass(frozen=True)
class TileLayout:
    """How zero-bordered channel tiles occupy ciphertext slots (conv.py:63-110).

    ring: rotation-orbit size (n direct, n/2 batch); units: orbits per
    ciphertext; c_n: tiles per orbit; frags/frag_len/halo: the split of a
    tile larger than one orbit into self-contained fragments."""

    n: int
    height: int
    width: int
    pad: int
    ring: int
    units: int
    c_n: int
    frags: int
    frag_len: int
    halo: int
    stride: int = 1

    @property
    def w_p(self) -> int:
        return self.width + 2 * self.pad

    @property
    def h_p(self) -> int:
        return self.height + 2 * self.pad

    @property
    def tile(self) -> int:
        return self.h_p * self.w_p

    @property
    def fragmented(self) -> bool:
        return self.frags > 1

    def units_for(self, channels: int) -> int:
        return channels * self.frags if self.fragmented else -(-channels // self.c_n)

    def ct_count(self, channels: int) -> int:
        return -(-self.units_for(channels) // self.units)

    def out_dims(self) -> tuple[int, int]:
        return self.height // self.stride, self.width // self.stride


def _make_layout(n: int, height: int, width: int, f_w: int, ring_slots: int, units: int) -> TileLayout:
    pad = f_w // 2
    tile = (height + 2 * pad) * (width + 2 * pad)
    common = dict(n=n, height=height, width=width, pad=pad, ring=ring_slots, units=units)
    if tile <= ring_slots:
        return TileLayout(**common, c_n=ring_slots // tile, frags=1, frag_len=tile, halo=0)
    halo = pad * (width + 2 * pad + 1)
    frag_len = ring_slots - 2 * halo
    if frag_len <= 0:
        raise ParameterError("ring too small for even one padded row window")
    return TileLayout(**common, c_n=1, frags=-(-tile // frag_len), frag_len=frag_len, halo=halo)


def layout_direct(params: RingParams, height: int, width: int, f_w: int) -> TileLayout:
    return _make_layout(params.n, height, width, f_w, params.n, 1)


def layout_batch(params: RingParams, height: int, width: int, f_w: int) -> TileLayout:
    return _make_layout(params.n, height, width, f_w, params.n // 2, 2)


@dataclass
class PackedTensor:
    cts: list[Ciphertext]
    layout: TileLayout
    channels: int
    scale: int = 0


# ---------------------------------------------------------------------------
# slot bookkeeping (host)


def _interior(layout: TileLayout, stride: int = 1) -> np.ndarray:
    """Row-major tile positions of the readable pixels (stride applied)."""
    h_out, w_out = layout.height // stride, layout.width // stride
    rows = layout.pad + stride * np.arange(h_out)
    cols = layout.pad + stride * np.arange(w_out)
    return (rows[:, None] * layout.w_p + cols[None, :]).reshape(-1)


def tile_vector(channel: np.ndarray, layout: TileLayout, p: int) -> np.ndarray:
    """One channel as a zero-bordered row-major tile, values mod p."""
    out = np.zeros(layout.tile, dtype=np.int64)
    out[_interior(layout)] = (np.asarray(channel, dtype=np.int64) % p).reshape(-1)
    return out


def channel_positions(layout: TileLayout, j: int) -> tuple[np.ndarray, np.ndarray]:
    """(ciphertext index, slot) of channel j's readable values (conv.py:162-177)."""
    tp = _interior(layout, layout.stride)
    if layout.fragmented:
        frag = tp // layout.frag_len
        unit = j * layout.frags + frag
        slot = (unit % layout.units) * layout.ring + layout.halo + tp - frag * layout.frag_len
        return unit // layout.units, slot
    unit = j // layout.c_n
    slot = (unit % layout.units) * layout.ring + layout.tile * (j % layout.c_n) + tp
    return np.full(tp.shape, unit // layout.units, dtype=np.int64), slot


def pack_vectors(values: np.ndarray, layout: TileLayout, p: int) -> list[np.ndarray]:
    """Slot vectors (length n) for a (c, H, W) integer tensor (conv.py:180-197)."""
    c = len(values)
    vecs = np.zeros((layout.ct_count(c), layout.n), dtype=np.int64)
    for j in range(c):
        tv = tile_vector(values[j], layout, p)
        if not layout.fragmented:
            unit = j // layout.c_n
            start = (unit % layout.units) * layout.ring + layout.tile * (j % layout.c_n)
            vecs[unit // layout.units, start : start + layout.tile] = tv
            continue
        for k in range(layout.frags):
            unit = j * layout.frags + k
            base = (unit % layout.units) * layout.ring
            first = k * layout.frag_len - layout.halo  # tile index of the orbit's slot 0
            lo, hi = max(first, 0), min(first + layout.ring, layout.tile)
            vecs[unit // layout.units, base + lo - first : base + hi - first] = tv[lo:hi]
    return list(vecs)


def pack_input(values, params: RingParams, f_w: int, encrypt_fn, batch: bool = False, scale: int = 0) -> PackedTensor:
    """Zero-bordered tiles, encoded and encrypted ciphertext by ciphertext."""
    values = np.asarray(values, dtype=np.int64)
    c, h, w = values.shape
    layout = (layout_batch if batch else layout_direct)(params, h, w, f_w)
    encode = bfv.encode_batch if batch else bfv.encode_direct
    cts = [encrypt_fn(encode(v, params)) for v in pack_vectors(values, layout, params.p)]
    if batch:
        cts = [bfv.to_eval(ct, params) for ct in cts]
    return PackedTensor(cts, layout, c, scale)


def pack_input_private(values, params: RingParams, f_w: int, sk: bfv.SecretKey, rng, scale: int = 0) -> PackedTensor:
    """pack_input with encrypt_fn = encrypt_private(·, sk, rng), the encryptions
    batched (bfv.encrypt_private_rows): bit-identical ciphertexts and RNG
    consumption, one device pass instead of one per ciphertext; the result is
    one device-resident stack."""
    values = np.asarray(values, dtype=np.int64)
    c, h, w = values.shape
    layout = layout_direct(params, h, w, f_w)
    msgs = np.stack([np.asarray(v, dtype=np.int64) for v in pack_vectors(values, layout, params.p)])
    return PackedTensor(bfv.encrypt_private_rows(msgs, sk, rng), layout, c, scale)


def unpack(tensor: PackedTensor, sk: bfv.SecretKey, signed: bool = True) -> np.ndarray:
    """Decrypt (batched on the device) and gather readable slots to (c, H', W')."""
    params = sk.params
    m, _ = bfv.decrypt_rows(tensor.cts, sk)
    if tensor.cts[0].encoding == Encoding.BATCH:
        ring.get_plan(params.n, params.p)
        m = ring.ntt_rows(m, params.n, [params.p])
        slots = m.cpu().numpy()[:, bfv._slot_index(params)]
    else:
        slots = m.cpu().numpy()
    h_out, w_out = tensor.layout.out_dims()
    out = np.zeros((tensor.channels, h_out * w_out), dtype=np.int64)
    for j in range(tensor.channels):
        ci, si = channel_positions(tensor.layout, j)
        out[j] = slots[ci, si]
    if signed:
        out = bfv.centered(out, params.p)
    return out.reshape(tensor.channels, h_out, w_out)


# ---------------------------------------------------------------------------
# K1 plans


def _tap_steps(layout: TileLayout, f_w: int) -> np.ndarray:
    """DRot step of each tap, row-major: (dy−pad)·W_p + (dx−pad) (conv.py:245-248)."""
    off = np.arange(f_w) - f_w // 2
    return (off[:, None] * layout.w_p + off[None, :]).reshape(-1)


def _check_budget(weights2d: np.ndarray):
    """max_o Σ|w| < 2^32 (conv.py:314-319, ring.py:344)."""
    if weights2d.size == 0:
        return
    worst = int(np.abs(weights2d).sum(axis=1).max())
    if worst >= ring.WEIGHT_BUDGET:
        raise AccumulatorBudgetError(f"layer needs |weight| sum {worst}, over the lazy accumulation budget")


class ConvPlan:
    """Device operands of one K1 contraction.

    out[o*frags + f][p] = Σ_k w[o, k] · in[src[k] + f·fstride][p] · x^(−step[k])
                          (+ Δ·bias[o] on the slots of mask[f], c0 only)
    """

    def __init__(self, q: int, n: int, weights2d: np.ndarray, src: np.ndarray, step: np.ndarray,
                 frags: int = 1, fstride: int = 0, bias_delta: np.ndarray | None = None,
                 bias_mask: np.ndarray | None = None):
        weights2d = np.asarray(weights2d, dtype=np.int64)
        if weights2d.size and int(np.abs(weights2d).max()) >= 1 << 15:
            raise ParameterError("K1 weights must fit int16")
        self.q, self.n = int(q), int(n)
        self.c_o, self.K = weights2d.shape
        self.frags, self.fstride = int(frags), int(fstride)
        step = np.asarray(step, dtype=np.int64)
        if step.size and (step.max() >= n or step.min() <= -n):
            raise ParameterError("DRot step outside (-n, n)")
        dev = device.require_cuda()
        self.w = torch.from_numpy(weights2d.astype(np.int16)).to(dev)
        self.src = torch.from_numpy(np.asarray(src, dtype=np.int32)).to(dev)
        self.step = torch.from_numpy(step.astype(np.int32)).to(dev)
        self.bias = None if bias_delta is None else torch.from_numpy(np.asarray(bias_delta, dtype=np.uint64).view(np.int64)).to(dev)
        self.mask = None if bias_mask is None else torch.from_numpy(np.asarray(bias_mask, dtype=np.uint8)).to(dev)
        self.n_out = self.c_o * self.frags
        self.tc: ConvTcPlan | None = None  # tensor-core variant, when the layer qualifies

    @property
    def path(self) -> str:
        return "tc" if self.tc is not None and _conv_path() != "int" else "int"

    def run(self, inp: torch.Tensor, out: torch.Tensor | None = None, path: str | None = None) -> torch.Tensor:
        """inp: device [n_in, 2, n] -> out [c_o*frags, 2, n]. `path` ("tc" |
        "int") overrides the variant choice (both give identical results)."""
        inp = inp.contiguous()
        if out is None:
            out = torch.empty((self.n_out, 2, self.n), dtype=torch.int64, device=inp.device)
        path = path or self.path
        if path == "tc" and self.tc is None:
            raise ParameterError("this layer has no tensor-core plan")
        if path == "tc":
            return self.tc.run(inp, out)
        _native.call(
            "fhe_conv_flash", self.q, self.n, inp.data_ptr(), inp.shape[0], self.w.data_ptr(), self.c_o, self.K,
            self.src.data_ptr(), self.step.data_ptr(), self.frags, self.fstride, device.ptr(self.bias),
            device.ptr(self.mask), out.data_ptr(), device.stream(),
        )
        return out


def _conv_path() -> str:
    """FLASHHE_CONV_PATH = auto (default) | int | tc — which K1 variant runs."""
    return _os.environ.get("FLASHHE_CONV_PATH", "auto")


class ConvTcPlan:
    """K1-TC operands (csrc/conv_tc.cu): packed int8 weights, the digit-plane
    operand buffer X and the tap steps. Eligible when |w| ≤ 127, 2^56 ≤ q,
    n a multiple of 64 and the halo window fits shared memory (input channels
    are zero-padded to a multiple of 32). GEMM tile: 128 output channels ×
    `pos_tile` positions."""

    OC_TILE = 128  # output channels per tile (tcgen05 M)
    SMS = 148  # B200 SM count (tile-size heuristic only)

    @staticmethod
    def _fits(pos_tile: int, h: int, taps: int) -> bool:
        win = -(-(pos_tile + 2 * h) * 256 // 1024) * 1024
        return 2 * (win + taps * ConvTcPlan.OC_TILE * 32) <= 218 * 1024  # >= 2 pipeline stages (csrc kRingBudget)

    @staticmethod
    def pos_tile_for(c_o: int, n: int, frags: int, h: int, taps: int, c_i: int = 32) -> int:
        """Positions per tile (csrc/conv_tc.cu): 32, 64 or 16. FLASHHE_TC_POS =
        auto (default) | 32 | 16 | 64. `auto` takes 64 (two accumulators share
        each weight stage: half the weight bytes per position, but no TMEM
        double buffering) for long contractions (ceil(c_i/32)·taps >= 72, the
        s3/s4 layers: measured 1.2 % faster on config 5 and 0.5 % on config 4
        with dynamic tile scheduling), 16 when 32 does not fit, else 32."""
        import os

        mode = os.environ.get("FLASHHE_TC_POS", "auto")
        if mode != "auto":
            return int(mode) if int(mode) <= 32 or ConvTcPlan._fits(int(mode), h, taps) else 32
        if not ConvTcPlan._fits(32, h, taps):
            return 16
        if -(-c_i // 32) * taps >= 72 and ConvTcPlan._fits(64, h, taps):
            return 64
        return 32

    @staticmethod
    def rep_for(c_o: int, JB: int, taps: int, h: int) -> tuple[int, int]:
        """(rep, 1): position groups stacked in the 128 accumulator rows
        (csrc/conv_tc.cu LayerDesc.rep). A layer with c_o <= 64 fills only
        c_o TMEM lanes, so only the warps of c_o/32 lane quadrants (SM
        sub-partitions) can read its accumulators: short contractions (JB·taps
        <= 16 MMAs per 32 positions — the stems) are then bound by the
        epilogue, not the MMAs. With rep groups, rows r·128/rep + o compute
        channel o at positions 32 r.. of the tile (the same window, tap offsets
        + 32 r): every quadrant's warps run the epilogue, for the same MMA work
        per position. FLASHHE_TC_REP (1 | 2 | 4) forces a rep where it is
        valid. (The second value is the C ABI's reserved tsplit field: a
        block's MMAs always run in one stage; a split over several stages was
        measured slower and removed.)"""
        import os

        def fit(r):
            stage = -(-(32 * r + 2 * h) * 256 // 1024) * 1024 + taps * r * 32 * ConvTcPlan.OC_TILE
            return 2 * stage <= 218 * 1024

        def ok(r):
            return r == 1 or (c_o <= ConvTcPlan.OC_TILE // r and taps * r <= 64 and fit(r))

        forced = os.environ.get("FLASHHE_TC_REP")
        if forced and ok(int(forced)):
            r = int(forced)
        elif forced or JB * taps > 16:
            r = 1
        else:
            r = next(r for r in (4, 2, 1) if ok(r))
        return r, 1

    @staticmethod
    def ilv_for(c_o: int, JB: int, steps, h: int, rep: int) -> list[int] | None:
        """The merged window offsets of an interleaved layer, or None when the
        layer keeps stacked groups. With c_o <= 64 half of every 128-row MMA is
        idle (rep 1) or zero (rep 2). Interleaving the two groups — row 2 o + r
        = channel o at positions 2 u + r, the window read at stride 2 — makes
        the taps with equal offset step + r ONE full MMA: the 7 column taps of
        the 7x7 stem take 8 MMAs per 64 positions instead of 14, a 3x3 layer 12
        instead of 18, and every TMEM lane quadrant has epilogue work.
        FLASHHE_TC_ILV = auto (default) | 0."""
        import os

        if os.environ.get("FLASHHE_TC_ILV", "auto") == "0" or c_o > 64 or rep > 2:
            return None
        st = [int(s) for s in steps]
        merged = sorted(set(st) | {s + 1 for s in st})
        if len(set(st)) != len(st) or len(merged) >= 2 * len(st) or len(merged) > 64:
            return None  # repeated steps, nothing to merge (e.g. 1x1), or above the kernel's tap limit
        stage = -(-(64 + 2 * h) * 256 // 1024) * 1024 + len(merged) * 32 * ConvTcPlan.OC_TILE
        return merged if 2 * stage <= 218 * 1024 else None

    @staticmethod
    def eligible(weights3d: np.ndarray, q: int, n: int, h: int, taps: int) -> bool:
        c_o, c_i, _ = weights3d.shape
        if n < 64 or n % 64 or taps > 64 or 2 * h >= n:
            return False
        if int(np.abs(weights3d).max(initial=0)) > 127:
            return False
        if 127 * 255 * (-(-c_i // 32) * 32) * taps >= 1 << 31:  # exact s32 plane sums
            return False
        if not (1 << 56) <= q < (1 << 62):  # single-offset epilogue reduction (csrc/conv_tc.cu)
            return False
        return ConvTcPlan._fits(16, h, taps)

    def __init__(self, q: int, n: int, weights3d: np.ndarray, steps: np.ndarray, layout: TileLayout | None,
                 bias, mask, chan: np.ndarray | None = None):
        """`chan` ([c_i, 2]: source ciphertext, slot offset) replaces the
        layout's channel placement — fully_connected's per-input DRot slots,
        or a tap-folded conv's (channel, tap) pairs (fragment f then reads
        source + f when the layout is fragmented)."""
        self.q, self.n = int(q), int(n)
        self.c_o, self.c_i, self.taps = weights3d.shape
        self.h = int(np.abs(steps).max(initial=0))
        self.frags = layout.frags if layout is not None else 1
        self.pos_tile = self.pos_tile_for(self.c_o, self.n, self.frags, self.h, self.taps, self.c_i)
        N = self.OC_TILE
        OB, JB = -(-self.c_o // N), -(-self.c_i // 32)
        self.rep, self.tsplit = self.rep_for(self.c_o, JB, self.taps, self.h) if self.pos_tile == 32 else (1, 1)
        j = np.arange(self.c_i)
        if chan is not None:
            chan = np.asarray(chan, dtype=np.int64).reshape(self.c_i, 2)
            self.fstride = 1 if layout is not None and layout.fragmented else 0
        elif layout.fragmented:
            chan, self.fstride = np.stack([j * layout.frags, np.zeros_like(j)], 1), 1
        else:
            chan, self.fstride = np.stack([j // layout.c_n, layout.tile * (j % layout.c_n)], 1), 0
        merged = self.ilv_for(self.c_o, JB, steps, self.h, self.rep) if self.pos_tile == 32 else None
        if merged is not None:
            # Interleaved position groups (csrc/conv_tc.cu LayerDesc.ilv): row 2 o + r computes channel o
            # at positions 2 u + r, so tap t of group r reads window offset step_t + r — taps of the two
            # groups with the same offset share one full-height MMA. The C layer sees the merged taps.
            self.rep, self.tsplit = 2, 2
            T = len(merged)
            wp = np.zeros((OB * N, JB * 32, T), dtype=np.int8)
            for r in range(2):
                for t, st in enumerate(steps):
                    wp[r : 2 * self.c_o : 2, : self.c_i, merged.index(int(st) + r)] = weights3d[:, :, t]
            steps = np.asarray(merged, dtype=np.int64)
        else:
            T = self.taps * self.rep
            wp = np.zeros((OB * N, JB * 32, T), dtype=np.int8)
            rows = N // self.rep
            for r in range(self.rep):  # position group r: rows [r·rows, r·rows + c_o), tap blocks [r·taps, (r+1)·taps)
                wp[r * rows : r * rows + self.c_o, : self.c_i, r * self.taps : (r + 1) * self.taps] = weights3d
        self.k_taps = len(steps)  # taps as the C layer counts them (merged when interleaved)
        # [ob][jb][tap][g][kh][r][jj] with o = ob*128 + g*8 + r, j = jb*32 + kh*16 + jj
        wp = wp.reshape(OB, N // 8, 8, JB, 2, 16, T).transpose(0, 3, 6, 1, 4, 2, 5)
        dev = device.require_cuda()
        self.w = torch.from_numpy(np.ascontiguousarray(wp)).to(dev)
        self.chan = torch.from_numpy(np.ascontiguousarray(chan, dtype=np.int32)).to(dev)
        self.steps = (ctypes.c_int32 * self.k_taps)(*[int(s) for s in steps])
        self.sync = device.zeros_i64(SYNC_WORDS)  # counters of this plan's own launches
        self._single: dict = {}  # cached one-layer launch arguments per (input, output) buffers
        self.bias, self.mask = bias, mask

    @property
    def x_bytes(self) -> int:
        """Size of the digit-plane operand X: [2][frags][JB][n + 2h][256 B]."""
        return 2 * self.frags * (-(-self.c_i // 32)) * (self.n + 2 * self.h) * 256

    def layer(self, inp: torch.Tensor, out: torch.Tensor, alone: bool = False) -> "_native.ConvTcLayer":
        """This layer's entry of a fhe_conv_tc_stack launch. `alone`: the layer is
        the launch's only one — 64-position tiles (chosen for a stack, where other
        layers fill the tail) then give way to 32-position ones: twice the tiles
        over the 148 CTAs (a config-5 s3 layer alone: 128 -> 256 tiles, 41 -> 28 us)."""
        pos_tile = 32 if alone and self.pos_tile == 64 and _os.environ.get("FLASHHE_TC_POS", "auto") == "auto" else self.pos_tile
        return _native.ConvTcLayer(
            inp.data_ptr(), inp.numel() // (2 * self.n), self.c_i, self.frags, self.fstride, self.chan.data_ptr(), self.h, self.w.data_ptr(),
            self.c_o, self.k_taps, pos_tile, ctypes.cast(self.steps, ctypes.c_void_p), device.ptr(self.bias),
            device.ptr(self.mask), out.data_ptr(), self.rep, self.tsplit)

    def run(self, inp: torch.Tensor, out: torch.Tensor, mark=None) -> torch.Tensor:
        """One cooperative persistent launch of this layer alone (relayout,
        grid barrier, tcgen05 GEMM); `mark()` (e.g. a CUDA event record) runs
        right before it when given. The launch arguments are cached per
        (input, output) buffer pair: a repeated call is one C call."""
        if mark is not None:
            mark()
        key = (inp.data_ptr(), inp.numel(), out.data_ptr())
        hit = self._single.get(key)
        if hit is None:
            if len(self._single) > 16:
                self._single.clear()
            need = _x_total([self])
            hit = self._single[key] = ((_native.ConvTcLayer * 1)(self.layer(inp, out, alone=True)), need)
        arr, need = hit
        X = device.scratch("conv_tc_x", need)
        rc = _stack_launch(self.q, self.n, arr, 1, X, 0, self.sync.data_ptr(), device.stream())
        if rc:
            _native.check(rc)
        return out


SYNC_WORDS = 3 + 4 * 24  # fhe_conv_tc_stack: launch counter + per-layer work / relayout-done / GEMM-done / tile counters
MAX_STACK = 24
_stack_sync: dict[tuple, torch.Tensor] = {}


def _stack_sync_for(tcs) -> torch.Tensor:
    """The counter buffer of one layer sequence (see run_tc_stack)."""
    key = (torch.cuda.current_device(),) + tuple(id(tc) for tc in tcs)
    sync = _stack_sync.get(key)
    if sync is None:
        sync = _stack_sync[key] = device.zeros_i64(SYNC_WORDS)
    return sync


def _x_total(tcs) -> int:
    """Digit-plane scratch of one launch: each layer's X region, 256-byte aligned."""
    return sum(-(-tc.x_bytes // 256) * 256 for tc in tcs)


def _stack_launch(*args) -> int:
    return _native.fn("fhe_conv_tc_stack")(*args)


def run_tc_stack(jobs, sync: torch.Tensor | None = None) -> None:
    """One fhe_conv_tc_stack launch for [(ConvTcPlan, inp, out)] (≤ 24 layers
    sharing q and n) on the current stream. `sync` defaults to a counter
    buffer cached per layer sequence (the kernel's counters only grow, so a
    buffer is tied to one stack length and must not serve concurrent launches)."""
    tc0 = jobs[0][0]
    if len(jobs) > MAX_STACK:
        raise ValueError(f"at most {MAX_STACK} layers per tensor-core launch")
    if sync is None:
        sync = _stack_sync_for([tc for tc, *_ in jobs])
    X = device.scratch("conv_tc_x", _x_total([tc for tc, *_ in jobs]))  # every layer its own operand region
    arr = (_native.ConvTcLayer * len(jobs))(*[tc.layer(inp, out, alone=len(jobs) == 1) for tc, inp, out in jobs])
    rc = _native.fn("fhe_conv_tc_stack")(tc0.q, tc0.n, arr, len(jobs), X, 0, sync.data_ptr(), device.stream())
    if rc:
        _native.check(rc)


_side_streams: dict[int, tuple] = {}


def _streams():
    """(upload, download) side streams of the current device."""
    dev = torch.cuda.current_device()
    st = _side_streams.get(dev)
    if st is None:
        st = _side_streams[dev] = (torch.cuda.Stream(), torch.cuda.Stream())
    return st


def issue_k1(items, on_gemm=None) -> list:
    """Enqueue K1 for independent jobs [(plan, inp, ready_event | None, out)]
    on the current stream. Consecutive tensor-core jobs (up to 24) share ONE
    fhe_conv_tc_stack launch — layer i+1 is relaid out while layer i's GEMM
    runs and no per-layer launch gap remains; other jobs run one launch each. `on_gemm(i, "start" | "end")` is called around every
    tensor-core launch (i = its first job; e.g. to record timing events).
    Returns one completion event per job (jobs of one launch share it),
    recorded on the current stream. CUDA-graph capturable."""
    comp = torch.cuda.current_stream()
    tcs = [plan.tc for plan, *_ in items if plan.path == "tc"]
    if tcs:  # size the operand buffers before anything is enqueued (covers every launch of the call)
        device.scratch("conv_tc_x", _x_total(tcs))
    done = [None] * len(items)
    i = 0
    while i < len(items):
        j = i + 1
        if items[i][0].path == "tc":
            while j < len(items) and j - i < MAX_STACK and items[j][0].path == "tc":
                j += 1
        for _, _, ready, _ in items[i:j]:
            if ready is not None:
                comp.wait_event(ready)
        if items[i][0].path == "tc":
            if on_gemm:
                on_gemm(i, "start")
            # Jobs of one launch are independent, so their order is free (see
            # _stack_schedule: the launch is a two-stage relayout -> GEMM pipeline).
            run = _stack_schedule(items[i:j]) if _stack_order() else items[i:j]
            run_tc_stack([(plan.tc, inp, out) for plan, inp, _, out in run])
            if on_gemm:
                on_gemm(i, "end")
        else:
            plan, inp, _, out = items[i]
            plan.run(inp, out)
        ev = torch.cuda.Event()
        ev.record(comp)
        done[i:j] = [ev] * (j - i)
        i = j
    return done


def _stack_order() -> bool:
    """FLASHHE_STACK_ORDER = johnson (default, _stack_schedule) | given."""
    import os

    return os.environ.get("FLASHHE_STACK_ORDER", "johnson") != "given"


# Rough per-layer stage times of a stacked K1-TC launch (B200, measured):
# relayout by the 4 relayout warps of every CTA ~0.9 TB/s of digit-plane
# operand; GEMM bounded by the int8 MMA rate (~4 POPS, 16 ops per 60-bit x
# 8-bit MAC) or by the epilogue's TMEM reads (32 B per output coefficient,
# ~9.5 TB/s over the chip), plus ~2 us of per-layer pipeline fill. A layer's
# relayout also has a ~4 us latency floor (first loads of a cold input, the
# completion fences and count): without it Johnson's rule put the small
# layers first and the GEMM waited on their relayouts (config 5 0.403 ->
# 0.390 ms, config 4 0.330 -> 0.316 ms with it; tools/order_search.py found
# no better order by measured local search). Dev knobs: FLASHHE_REL_FILL_US,
# FLASHHE_REL_TBPS, FLASHHE_GEMM_FILL_US.
_RELAYOUT_BPS, _MMA_OPS, _TMEM_BPS, _LAYER_FILL_S = 0.9e12, 4.0e15, 9.5e12, 2e-6
_RELAYOUT_FILL_S = float(_os.environ.get("FLASHHE_REL_FILL_US", "4")) * 1e-6
_RELAYOUT_BPS = float(_os.environ.get("FLASHHE_REL_TBPS", "0.9")) * 1e12
_LAYER_FILL_S = float(_os.environ.get("FLASHHE_GEMM_FILL_US", "2")) * 1e-6


def _stage_times(plan: "ConvPlan") -> tuple[float, float]:
    tc = plan.tc
    macs = plan.n_out * plan.K * 2 * plan.n
    gemm = max(16 * macs / _MMA_OPS, plan.n_out * 2 * plan.n * 32 / _TMEM_BPS) + _LAYER_FILL_S
    return tc.x_bytes / _RELAYOUT_BPS + _RELAYOUT_FILL_S, gemm


def _stack_schedule(items):
    """Order of the independent jobs of one stacked launch. The launch is a
    two-stage pipeline — every job is relaid out (stage 1, relayout warps, in
    order) and then multiplied (stage 2, the GEMM roles, in order, each job
    once its operand is complete) — so Johnson's rule for the two-machine
    flow shop minimises the makespan: jobs whose relayout is shorter than
    their GEMM first, by increasing relayout time; then the others, by
    decreasing GEMM time. Stable for equal keys."""
    times = [_stage_times(it[0]) for it in items]
    first = sorted((k for k, (r, g) in enumerate(times) if r < g), key=lambda k: times[k][0])
    last = sorted((k for k, (r, g) in enumerate(times) if r >= g), key=lambda k: -times[k][1])
    return [items[k] for k in first + last]


def conv_plan(layer: ConvLayerSpec, layout: TileLayout, params: RingParams) -> ConvPlan:
    """K1 operands of conv_proposed for `layer` on `layout`, cached on the layer
    object (weights are treated as immutable after first use)."""
    key = (layout, params.fingerprint())
    cache = layer.__dict__.setdefault("_k1_plans", {})
    if key in cache:
        return cache[key]
    _check_budget(layer.weights.reshape(layer.c_o, -1))
    taps = layer.f_w * layer.f_w
    steps = _tap_steps(layout, layer.f_w)
    j = np.repeat(np.arange(layer.c_i), taps)
    t = np.tile(np.arange(taps), layer.c_i)
    if layout.fragmented:
        src, fstride, step = j * layout.frags, 1, steps[t]
    else:
        src, fstride, step = j // layout.c_n, 0, steps[t] + layout.tile * (j % layout.c_n)
    out_layout = replace(layout, c_n=1)
    bias_delta = bias_mask = None
    if layer.bias is not None and np.any(layer.bias):
        bias_delta = np.array([params.delta * (int(b) % params.p) % params.q for b in layer.bias], dtype=np.uint64)
        bias_mask = np.stack([_bias_mask(out_layout, f) for f in range(layout.frags)])
    plan = ConvPlan(params.q, params.n, layer.weights.reshape(layer.c_o, -1), src, step,
                    frags=layout.frags, fstride=fstride, bias_delta=bias_delta, bias_mask=bias_mask)
    h = int(np.abs(steps).max(initial=0))
    fold = _tap_fold(layer.c_i, layer.f_w)
    if fold == "none":
        if ConvTcPlan.eligible(layer.weights, params.q, params.n, h, taps):
            plan.tc = ConvTcPlan(params.q, params.n, layer.weights, steps, layout, plan.bias, plan.mask)
    else:
        # Few input channels (the stems): move taps into the contraction.
        # "full": virtual channel (j, t) = channel j read at tap t's DRot
        #   offset; one tap, no halo (3x3 stems: 27 channels, one MMA per stage).
        # "rows": virtual channel (j, dy) = channel j read at row dy's offset
        #   (dy - pad)·W_p; the f_w column taps stay descriptor offsets (halo
        #   pad). The 7x7 stem folds 21 channels into ONE 32-channel block
        #   instead of 147 into five: the digit-plane operand X is 5x smaller.
        c_i, f, pad = layer.c_i, layer.f_w, layer.f_w // 2
        if fold == "full":
            v_steps, t_steps = steps, np.zeros(1, dtype=np.int64)
            w3 = layer.weights.reshape(layer.c_o, c_i * taps, 1)
        else:
            v_steps, t_steps = (np.arange(f) - pad) * layout.w_p, np.arange(f) - pad
            w3 = layer.weights.reshape(layer.c_o, c_i * f, f)
        nv = len(v_steps)
        jj, tt = np.repeat(np.arange(c_i), nv), np.tile(np.arange(nv), c_i)
        if layout.fragmented:
            chan = np.stack([jj * layout.frags, v_steps[tt]], 1)
        else:
            chan = np.stack([jj // layout.c_n, layout.tile * (jj % layout.c_n) + v_steps[tt]], 1)
        th = int(np.abs(t_steps).max(initial=0))
        if ConvTcPlan.eligible(w3, params.q, params.n, th, len(t_steps)):
            plan.tc = ConvTcPlan(params.q, params.n, w3, t_steps, layout, plan.bias, plan.mask, chan=chan)
    cache[key] = plan
    return plan


def _tap_fold(c_i: int, f_w: int) -> str:
    """How K1-TC lays out a layer's taps: "none" (channels in 32-wide blocks,
    all taps as DRot descriptor offsets), "rows" or "full" (taps folded into
    virtual channels). Fewest 32-channel blocks first (each block is one
    digit-plane slab of X, written once and streamed by the GEMM), then the
    fewest MMAs per tile (blocks x remaining taps)."""
    taps = f_w * f_w
    if taps == 1:
        return "none"
    cand = {"none": (-(-c_i // 32), taps), "rows": (-(-(c_i * f_w) // 32), f_w), "full": (-(-(c_i * taps) // 32), 1)}
    return min(cand, key=lambda k: (cand[k][0], cand[k][0] * cand[k][1]))


def _bias_mask(layout: TileLayout, frag: int) -> np.ndarray:
    """Slots where conv.py:_bias_plaintext (414-424) places the bias value."""
    mask = np.zeros(layout.n, dtype=np.uint8)
    tp = _interior(layout)
    if layout.fragmented:
        tp = tp[tp // layout.frag_len == frag]
        mask[layout.halo + tp - frag * layout.frag_len] = 1
    else:
        mask[tp] = 1
    return mask


def conv_proposed(x: PackedTensor, layer: ConvLayerSpec, params: RingParams, lazy: bool = True,
                  workers: int = 1, out: torch.Tensor | None = None) -> PackedTensor:
    """Algorithm 1 (conv.py:355-411) as one K1 launch: every output channel
    and fragment at once, one modular reduction per coefficient. `lazy` and
    `workers` are accepted for API compatibility; the result is the same
    canonical ciphertext either way (as in the reference). `out` (addition):
    a device [c_o·frags, 2, n] int64 buffer the result is written into — a
    caller running the same layer repeatedly (inference.he_forward) reuses
    one buffer instead of a fresh large allocation per call."""
    plan = _proposed_plan(x, layer, params)
    if out is not None and (tuple(out.shape) != (plan.n_out, 2, params.n) or out.dtype != torch.int64
                            or not out.is_contiguous()):
        raise ParameterError(f"out must be a contiguous int64 [{plan.n_out}, 2, {params.n}] tensor")
    out = plan.run(bfv.cts_rows(x.cts), out)
    cts = bfv.cts_from_rows(out, params.q, Encoding.DIRECT, Domain.COEFF)
    return PackedTensor(cts, _out_layout(x.layout), layer.c_o, x.scale + layer.weight_scale)


def conv_proposed_many(xs, layer: ConvLayerSpec, params: RingParams, outs=None) -> list[PackedTensor]:
    """conv_proposed over several independent inputs of ONE layer — e.g. the
    same layer of several inference requests (inference.he_forward_many).
    The tensor-core jobs run as stacked launches (issue_k1: up to 24 jobs in
    one fhe_conv_tc_stack launch, sharing the layer's packed weights), so the
    per-launch relayout latency and launch overhead of the one-job drop-in
    call are paid once per stack. `outs` (optional): one device output buffer
    per input, as conv_proposed's `out=`. Results equal conv_proposed's."""
    xs = list(xs)
    if not xs:
        return []
    items = []
    for i, x in enumerate(xs):
        plan = _proposed_plan(x, layer, params)
        out = outs[i] if outs is not None else None
        if out is not None and (tuple(out.shape) != (plan.n_out, 2, params.n) or out.dtype != torch.int64
                                or not out.is_contiguous()):
            raise ParameterError(f"out must be a contiguous int64 [{plan.n_out}, 2, {params.n}] tensor")
        inp = bfv.cts_rows(x.cts).contiguous()
        if out is None:
            out = torch.empty((plan.n_out, 2, params.n), dtype=torch.int64, device=inp.device)
        items.append((plan, inp, None, out))
    issue_k1(items)
    return [PackedTensor(bfv.cts_from_rows(out, params.q, Encoding.DIRECT, Domain.COEFF), _out_layout(x.layout),
                         layer.c_o, x.scale + layer.weight_scale) for x, (_, _, _, out) in zip(xs, items)]


_out_layouts: dict = {}


def _out_layout(layout: TileLayout) -> TileLayout:
    """replace(layout, c_n=1), cached (the conv output layout)."""
    o = _out_layouts.get(layout)
    if o is None:
        o = _out_layouts[layout] = replace(layout, c_n=1)
    return o


def _proposed_plan(x: PackedTensor, layer: ConvLayerSpec, params: RingParams) -> ConvPlan:
    layout = x.layout
    if (layout.height, layout.width) != (layer.height, layer.width) or layout.pad != layer.f_w // 2:
        raise ParameterError("tensor layout does not match the layer geometry")
    if layout.stride != 1:
        raise ParameterError("convolution input must not carry a pending stride")
    enc = x.cts.encoding if isinstance(x.cts, bfv.CtStack) else x.cts[0].encoding  # (no Ciphertext view built)
    if enc != Encoding.DIRECT:
        raise EncodingError("proposed convolution needs direct-encoded input")
    return conv_plan(layer, layout, params)  # runs _check_budget before caching a plan


def _stream_order(meta, params: RingParams) -> list[int]:
    """Issue order of conv_proposed_stream's independent jobs (results keep the
    call's order). The three streams form an upload -> K1 -> download pipeline
    whose downloads dominate (outputs are c_o·frags ciphertexts, inputs c_i·frags
    / c_n): the job with the smallest upload goes first, so the download stream
    starts early, and the job with the largest download second, so every other
    job's upload and convolution runs under it; the rest keep their order."""
    if len(meta) < 3 or _os.environ.get("FLASHHE_STREAM_ORDER") == "given":
        return list(range(len(meta)))
    n_in = [len(x.cts) for x, _, _ in meta]
    n_out = [plan.n_out for *_, plan in meta]
    first = min(range(len(meta)), key=lambda j: (n_in[j], n_out[j], j))
    rest = [j for j in range(len(meta)) if j != first]
    second = max(rest, key=lambda j: (n_out[j], -j))
    return [first, second] + [j for j in rest if j != second]


def conv_proposed_stream(jobs, params: RingParams) -> list[PackedTensor]:
    """Serving form of conv_proposed over a sequence of independent
    (PackedTensor, ConvLayerSpec) jobs — e.g. one layer of many requests, or
    many layers' pending inputs. Uploads, K1 launches and downloads run on
    three CUDA streams, so job i+1's upload and job i-1's download overlap
    job i's convolution.

    Inputs may be host- (ideally pinned, see bfv.cts_from_host) or device-
    resident. Outputs are canonical ciphertexts resident on both sides: the
    host copies (pinned) are complete when this returns. Results are exactly
    those of conv_proposed on each job."""
    device.require_cuda()
    comp = torch.cuda.current_stream()
    up, down = _streams()
    up.wait_stream(comp)
    meta = [(x, layer, _proposed_plan(x, layer, params)) for x, layer in jobs]  # validate before enqueueing
    need = -(-max((plan.tc.x_bytes for *_, plan in meta if plan.path == "tc"), default=0) // 256) * 256
    if need:  # sized once, before any job is enqueued (every job is a one-layer launch)
        device.scratch("conv_tc_x", need)
    # all of the call's host outputs in one pinned allocation (one allocator call, not one per job)
    sizes = [plan.n_out * 2 * params.n for *_, plan in meta]
    host_all = torch.empty(sum(sizes), dtype=torch.int64, pin_memory=True)
    views = torch.split(host_all, sizes)
    outs = [None] * len(meta)
    fast = _native.fn("fhe_conv_stream_job")
    ev_up, ev_comp = torch.cuda.Event(), torch.cuda.Event()
    ev_up.record(comp)  # create the cudaEvent handles (torch makes them on first record)
    ev_comp.record(comp)
    for j in _stream_order(meta, params):  # one pass: job i's download is enqueued before job i+1's upload
        (x, layer, plan), hv = meta[j], views[j]
        ready = None
        rows_in = x.cts.rows if isinstance(x.cts, bfv.CtStack) else None
        if plan.path == "tc" and rows_in is not None and rows_in._dev is None and rows_in._pinned is not None:
            # host-resident pinned input: upload, K1 and download in one C call (one
            # ctypes crossing per job instead of ~10 torch/ctypes calls)
            pin = rows_in._pinned
            # inp is written by the upload stream: allocate it there (its block is
            # then never handed out while a pending copy on `up` could still write
            # it) and tell the allocator the compute stream reads it
            with torch.cuda.stream(up):
                inp = torch.empty((pin.numel() // (2 * params.n), 2, params.n), dtype=torch.int64,
                                  device=comp.device)
            inp.record_stream(comp)
            out = torch.empty((plan.n_out, 2, params.n), dtype=torch.int64, device=comp.device)
            lay = (_native.ConvTcLayer * 1)(plan.tc.layer(inp, out, alone=True))
            sync = _stack_sync_for([plan.tc])
            X = device.scratch("conv_tc_x", need)  # already sized: never reallocated here
            rc = fast(params.q, params.n, lay, pin.data_ptr(), pin.numel() * 8, hv.data_ptr(), hv.numel() * 8, X,
                      need, sync.data_ptr(), up.cuda_stream, comp.cuda_stream, down.cuda_stream,
                      ev_up.cuda_event, ev_comp.cuda_event)
            if rc:
                _native.check(rc)
            rows_in._dev = inp.reshape(-1, params.n)
            h = hv.view(out.shape[0] * 2, params.n).numpy()
            h.flags.writeable = False
            rows = device.DeviceRows(dev=out.reshape(-1, params.n), host=h, pinned=hv)
            cts = bfv.CtStack(rows, params.q, Encoding.DIRECT, Domain.COEFF)
            outs[j] = PackedTensor(cts, replace(x.layout, c_n=1), layer.c_o, x.scale + layer.weight_scale)
            continue
        if isinstance(x.cts, bfv.CtStack):
            inp, ready = x.cts.rows.upload_on(up)
        else:
            inp = bfv.cts_rows(x.cts).reshape(-1, params.n)
        inp = inp.reshape(-1, 2, params.n)
        out = torch.empty((plan.n_out, 2, params.n), dtype=torch.int64, device=inp.device)
        (ev,) = issue_k1([(plan, inp, ready, out)])
        inp.record_stream(comp)
        down.wait_event(ev)
        rows = device.DeviceRows.download_on(out, down, into=hv)
        cts = bfv.CtStack(rows, params.q, Encoding.DIRECT, Domain.COEFF)
        outs[j] = PackedTensor(cts, replace(x.layout, c_n=1), layer.c_o, x.scale + layer.weight_scale)
    down.synchronize()
    return outs


def _bias_plaintext(layout: TileLayout, frag: int, value: int, params: RingParams):
    vec = _bias_mask(layout, frag).astype(np.int64) * (value % params.p)
    return bfv.encode_direct(vec, params)


# ---------------------------------------------------------------------------
# pooling and fully connected (conv.py:604-668) on K1


_fc_plans: dict[tuple, tuple] = {}


def residual_add(y: PackedTensor, shortcut: PackedTensor, params: RingParams, inplace: bool = True) -> PackedTensor:
    """ResNet shortcut addition on ciphertexts (addition; the reference has no
    model module): y, a conv_proposed output (one channel per ciphertext),
    plus `shortcut` in y's layout. `shortcut` is either another conv output
    (a projection) or the packed block input itself, whose channel j is moved
    from tile j mod c_n of ciphertext j / c_n to slot 0 by a DRot
    (bfv.drot, key-switch-free) and added (bfv.hadd) — one fhe_residual_add
    launch for the whole tensor. Written into y's rows when `inplace`."""
    sl = shortcut.layout
    if y.channels != shortcut.channels or y.layout.stride != 1 or sl.stride != 1:
        raise EncodingError("residual operands differ in channels or carry a pending stride")
    if replace(sl, c_n=1) != y.layout:
        raise EncodingError("shortcut layout does not match the conv output layout")
    c_n, tile = (1, 0) if sl.fragmented else (sl.c_n, sl.tile)
    yr, ar = bfv.cts_rows(y.cts).contiguous(), bfv.cts_rows(shortcut.cts).contiguous()
    count = yr.shape[0]
    if count != y.layout.ct_count(y.channels) or ar.shape[0] != -(-count // c_n) or ar.shape[0] != len(shortcut.cts):
        raise EncodingError("residual operands do not match their layouts")
    out = yr if inplace else torch.empty_like(yr)
    _native.call("fhe_residual_add", params.q, count, c_n, tile, params.n, yr.data_ptr(), ar.data_ptr(),
                 out.data_ptr(), device.stream())
    cts = bfv.cts_from_rows(out, params.q, Encoding.DIRECT, Domain.COEFF)
    return PackedTensor(cts, y.layout, y.channels, y.scale)


def avg_pool(x: PackedTensor, k: int, params: RingParams) -> PackedTensor:
    """k×k sliding sums via DRot taps of weight 1; /k² and the subsample are
    deferred (stride marker), as conv.py:604-623. One separable pass
    (fhe_avg_pool: 2k adds per slot, exact mod q, identical ciphertexts)."""
    layout = x.layout
    if layout.height % k or layout.width % k:
        raise ParameterError(f"pool size {k} does not divide {layout.height}×{layout.width}")
    if layout.stride != 1:
        raise ParameterError("pooling input must not carry a pending stride")
    if layout.fragmented and (k - 1) * (layout.w_p + 1) > layout.halo:
        raise ParameterError("pool window exceeds the fragment halo")
    inp = bfv.cts_rows(x.cts).contiguous()
    out = torch.empty_like(inp)
    _native.call("fhe_avg_pool", params.q, params.n, 2 * len(x.cts), k, layout.w_p, inp.data_ptr(), out.data_ptr(),
                 device.stream())
    cts = bfv.cts_from_rows(out, params.q, x.cts[0].encoding, Domain.COEFF)
    return PackedTensor(cts, replace(layout, stride=k), x.channels, x.scale)


def fully_connected(x: PackedTensor, weights: np.ndarray, params: RingParams, bias: np.ndarray | None = None,
                    weight_scale: int = 0) -> list[Ciphertext]:
    """Matrix-vector product: output row o = Σ_v W[o,v]·DRot(ct(v), slot(v)),
    the dot product landing in slot 0 (conv.py:626-668)."""
    plan = _fc_plan(x, weights, params, bias)
    out = plan.run(bfv.cts_rows(x.cts))
    return bfv.cts_from_rows(out, params.q, Encoding.DIRECT, Domain.COEFF)


def _fc_plan(x: PackedTensor, weights, params: RingParams, bias) -> ConvPlan:
    """K1 operands of fully_connected, cached per weight array object (as
    conv_plan caches per layer: weights are treated as immutable after first
    use) and input geometry."""
    import weakref

    key = (id(weights), x.layout, x.channels, params.fingerprint(),
           None if bias is None else np.asarray(bias, dtype=np.int64).tobytes())
    hit = _fc_plans.get(key)
    if hit is not None and hit[0]() is weights:
        return hit[1]
    plan = _build_fc_plan(x, weights, params, bias)
    try:
        ref = weakref.ref(weights)
    except TypeError:  # lists and other non-weakref-able containers: no caching
        return plan
    _fc_plans[key] = (ref, plan)
    weakref.finalize(weights, _fc_plans.pop, key, None)
    return plan


def _build_fc_plan(x: PackedTensor, weights, params: RingParams, bias) -> ConvPlan:
    weights = np.asarray(weights, dtype=np.int64)
    c_out, v_in = weights.shape
    if weights.size and int(np.abs(weights).max()) >= 1 << MAX_WEIGHT_BITS:
        raise ParameterError("fc weights exceed the lazy-reduction bound")
    pos = [channel_positions(x.layout, j) for j in range(x.channels)]
    ct_idx = np.concatenate([p[0] for p in pos])
    slots = np.concatenate([p[1] for p in pos])
    if len(slots) != v_in:
        raise ParameterError(f"weight matrix expects {v_in} inputs, tensor has {len(slots)}")
    _check_budget(weights)
    bias_delta = bias_mask = None
    if bias is not None and np.any(bias):
        bias_delta = np.array([params.delta * (int(b) % params.p) % params.q for b in bias], dtype=np.uint64)
        bias_mask = np.zeros((1, params.n), dtype=np.uint8)
        bias_mask[0, 0] = 1
    plan = ConvPlan(params.q, params.n, weights, ct_idx, slots, bias_delta=bias_delta, bias_mask=bias_mask)
    w3 = weights.reshape(c_out, v_in, 1)
    if ConvTcPlan.eligible(w3, params.q, params.n, 0, 1):
        # one tap, the DRot slot of each input as its channel offset (K1-TC)
        plan.tc = ConvTcPlan(params.q, params.n, w3, np.zeros(1, dtype=np.int64), None, plan.bias, plan.mask,
                             chan=np.stack([ct_idx, slots], 1))
    return plan


def read_scalar_outputs(cts: list[Ciphertext], sk: bfv.SecretKey) -> np.ndarray:
    """Slot-0 values of per-output ciphertexts, centered."""
    m, _ = bfv.decrypt_rows(cts, sk)
    return bfv.centered(m[:, 0].cpu().numpy(), sk.params.p)


# ---------------------------------------------------------------------------
# conventional baseline: HRot + PMult on batch-encoded tiles (conv.py:427-597)


def conventional_steps(layer: ConvLayerSpec, params: RingParams) -> list[int]:
    """Distinct rotation steps the baseline engine needs (conv.py:431-446)."""
    layout = layout_batch(params, layer.height, layer.width, layer.f_w)
    taps = _tap_steps(layout, layer.f_w)
    shifts = [0] if layout.fragmented else range(1 - layout.c_n, layout.c_n)
    steps = {int((t + d * layout.tile) % layout.ring) for d in shifts for t in taps}
    steps.discard(0)
    if not layout.fragmented and layout.units > 1:
        if max(layout.units_for(layer.c_i), layout.units_for(layer.c_o)) > 1:
            steps.add(bfv.COLUMN_ROTATION)
    return sorted(steps)


def _uniform_prepared(value: int, params: RingParams) -> bfv.PreparedPlaintext:
    """Every slot = value: a constant polynomial, whose NTT is constant."""
    v = int(value) % params.p
    if v > params.p // 2:
        v -= params.p
    return bfv.PreparedPlaintext(np.full(params.n, v % params.q, dtype=np.int64))


def _rotations(cts, needed, swks, params) -> tuple[torch.Tensor, dict]:
    """All rotations the baseline needs, batched: one digit pass per source
    set (hoisted, bfv.py:485-491) and one K4 launch per (step, swap) over
    every input ciphertext. Returns rows [nR, 2, n] (EVAL) and a map
    (b, step, swap) -> row."""
    n, q = params.n, params.q
    T = swks.decomp_log
    l = -(-q.bit_length() // T)
    B = len(cts)
    base = bfv.cts_rows(cts).reshape(B, 2, n)
    groups = sorted(needed)  # (step, swap)
    srcs = {False: base}
    if any(sw for _, sw in groups):
        digits = bfv.key_digits_rows(base[:, 1], params, T, l)
        srcs[True] = bfv.keyswitch_rows(base, digits, bfv.COLUMN_ROTATION, swks)
        ring._bump("modmul", 2 * n * l * B)
    digs = {}
    index = {}
    R = torch.empty((len(groups) * B, 2, n), dtype=torch.int64, device=base.device)
    for g, (step, swap) in enumerate(groups):
        src = srcs[swap]
        dst = R[g * B : (g + 1) * B]
        if step == 0:
            _copy_rows(dst, src)
        else:
            if swap not in digs:
                digs[swap] = bfv.key_digits_rows(src[:, 1], params, T, l)
            bfv.keyswitch_rows(src, digs[swap], step, swks, out=dst)
            ring._bump("modmul", 2 * n * l * B)
        for b in range(B):
            index[(b, step, swap)] = g * B + b
    return R, index


def _copy_rows(dst: torch.Tensor, src: torch.Tensor) -> None:
    """Contiguous device copy (one D2D memcpy on the current stream)."""
    src = src.contiguous()
    _native.call("fhe_copy_2d", dst.data_ptr(), src.numel() * 8, src.data_ptr(), src.numel() * 8, src.numel() * 8, 1,
                 device.stream())


def _stacked_keys(swks: bfv.SwitchingKeySet, steps: tuple) -> torch.Tensor:
    """[len(steps)][l][2][n] Montgomery keys of several steps, cached on the key set."""
    cache = swks.__dict__.setdefault("_stacked", {})
    t = cache.get(steps)
    if t is None:
        keys = [swks.device_keys(s) for s in steps]
        t = cache[steps] = torch.empty((len(keys),) + tuple(keys[0].shape), dtype=torch.int64, device=keys[0].device)
        for i, k in enumerate(keys):
            _copy_rows(t[i], k)
    return t


def _conventional_fused(in_cts, plan, swks, params, out) -> None:
    """HRot x PMult x HAdd of every output in one fhe_rot_pmac pass: each
    rotation (source ciphertext, step) is key-switched in registers from the
    hoisted digits and applied to every plaintext that uses it; rotated
    ciphertexts are never materialised (north_star b). The column-swap source
    set (packed layouts with two orbits) is one hoisted HRot of the inputs.
    The static operands (groups, term lists, plaintexts, stacked keys) are
    built once per (plan, key set, input count) and kept on the device."""
    n, q = params.n, params.q
    T = swks.decomp_log
    l = -(-q.bit_length() // T)
    B = len(in_cts)
    terms = plan["terms"]
    st_key = (id(swks), B)
    hit = plan["dev"].get(st_key)
    if hit is None or hit[0] is not swks:
        needed = {(st, sw) for tl in terms for _, st, sw, _ in tl}
        steps = tuple(sorted({st for st, _ in needed if st}))
        kidx = {st: i for i, st in enumerate(steps)}
        # rotation groups, ordered by key so consecutive groups reuse it from L2
        gkeys = sorted({(kidx.get(st, -1), int(sw) * B + b, st) for tl in terms for b, st, sw, _ in tl})
        gpos = {(src, st): g for g, (_, src, st) in enumerate(gkeys)}
        G = len(gkeys)
        tiles = -(-len(terms) // 16)
        per = [[[] for _ in range(G)] for _ in range(tiles)]
        for o, tl in enumerate(terms):
            for b, st, sw, p_ in tl:
                per[o // 16][gpos[(int(sw) * B + b, st)]].append((o % 16, p_))
        toff = np.zeros((tiles, G + 1), dtype=np.int32)
        flat = []
        for t in range(tiles):
            toff[t, 0] = len(flat)
            for g in range(G):
                flat.extend(per[t][g])
                toff[t, g + 1] = len(flat)
        garr = np.array([(src, k) for k, src, _ in gkeys], dtype=np.int32).reshape(-1, 2)
        gp = np.array([bfv._galois_element(st, n) if st else 1 for _, _, st in gkeys], dtype=np.uint64)
        tarr = np.asarray(flat, dtype=np.int32).reshape(-1, 2) if flat else np.zeros((1, 2), np.int32)
        pt_rows = plan["pt_rows"]
        assert tarr[:, 1].max(initial=0) < len(pt_rows)
        pt = device.to_device(np.stack(pt_rows))
        pt_mont = torch.empty_like(pt)
        _native.call("fhe_to_montgomery", _native.u64_array([q]), 1, 1, len(pt_rows), n, pt.data_ptr(),
                     pt_mont.data_ptr(), device.stream())
        dev = pt.device
        K = _stacked_keys(swks, steps) if steps else device.zeros_i64(1)
        st = {
            "swap": any(sw for _, sw in needed), "G": G, "tiles": tiles, "K": K, "pt": pt, "pt_mont": pt_mont,
            "g": torch.from_numpy(garr).to(dev), "gp": torch.from_numpy(gp.view(np.int64)).to(dev),
            "toff": torch.from_numpy(toff).to(dev), "terms": torch.from_numpy(np.ascontiguousarray(tarr)).to(dev),
            "rotations": sum(1 for k, _, _ in gkeys if k >= 0), "macs": len(flat),
        }
        plan["dev"][st_key] = hit = (swks, st)
    st = hit[1]
    ring._bump("modmul", 2 * n * (l * st["rotations"] + st["macs"]))
    base = bfv.cts_rows(in_cts).reshape(B, 2, n)
    nsrc = 2 if st["swap"] else 1
    D = torch.empty((nsrc * B, l, n), dtype=torch.int64, device=base.device)  # digits of every source set
    bfv.key_digits_rows(base[:, 1], params, T, l, out=D[:B])
    if st["swap"]:  # src = swap * B + b: the inputs, then their column swaps
        C = torch.empty((2 * B, 2, n), dtype=torch.int64, device=base.device)
        _copy_rows(C[:B], base)
        bfv.keyswitch_rows(base, D[:B], bfv.COLUMN_ROTATION, swks, out=C[B:])
        ring._bump("modmul", 2 * n * l * B)
        bfv.key_digits_rows(C[B:, 1], params, T, l, out=D[B:])
    else:
        C = base.contiguous()
    n_out, G, tiles = len(terms), st["G"], st["tiles"]
    chunks = max(1, min(G, -(-2 * 148 // ((n // 64) * tiles))))
    part = torch.empty((chunks, n_out, 2, n), dtype=torch.int64, device=C.device) if chunks > 1 else None
    _native.call("fhe_rot_pmac", q, n, l, C.data_ptr(), D.data_ptr(), st["K"].data_ptr(), G, st["g"].data_ptr(),
                 st["gp"].data_ptr(), n_out, st["toff"].data_ptr(), st["terms"].data_ptr(), st["pt_mont"].data_ptr(),
                 chunks, device.ptr(part), out.data_ptr(), device.stream())


def _conventional_plan(layer: ConvLayerSpec, layout: TileLayout, n_in: int, params: RingParams) -> dict:
    """The baseline's terms per output [(b, step, swap, plaintext row)], the
    encoded-weight plaintexts and the bias slots (conv.py:457-564), built once
    per (layer, layout) and cached on the layer (weights immutable after use)."""
    key = ("conventional", layout, n_in, params.fingerprint())
    cache = layer.__dict__.setdefault("_k1_plans", {})
    if key in cache:
        return cache[key]
    taps = _tap_steps(layout, layer.f_w)
    n, cpu, ring_slots = params.n, layout.c_n, params.n // 2
    in_cts = range(n_in)
    pts: dict[bytes, int] = {}

    pt_rows: list[np.ndarray] = []

    def pt_uniform(w: int) -> int:  # _uniform_prepared: constant polynomial, constant NTT
        key = b"u" + int(w).to_bytes(8, "little", signed=True)
        if key not in pts:
            v = int(w) % params.p
            if v > params.p // 2:
                v -= params.p
            pts[key] = len(pt_rows)
            pt_rows.append(np.full(n, v % params.q, dtype=np.int64))
        return pts[key]

    def pt_blocks(bw: np.ndarray) -> int:
        key = b"b" + bw.tobytes()
        if key not in pts:
            vec = np.zeros(n, dtype=np.int64)
            for (unit_in, blk), w in np.ndenumerate(bw):
                start = unit_in * layout.ring + blk * layout.tile
                vec[start : start + layout.tile] = w % params.p
            pts[key] = len(pt_rows)
            pt_rows.append(bfv.prepare_plaintext(bfv.encode_batch(vec, params), params).evals)
        return pts[key]

    terms: list[list[tuple]] = []  # per output: [(b, step, swap, pt)]
    biases = []
    if layout.fragmented:
        pairs = -(-layout.frags // layout.units)
        for oc in range(layer.c_o):
            for t in range(pairs):
                tl = []
                for j in range(layer.c_i):
                    b = j * pairs + t
                    for k, step in enumerate(taps):
                        w = int(layer.weights[oc, j, k])
                        if w:
                            tl.append((b, int(step) % ring_slots, False, pt_uniform(w)))
                terms.append(tl)
                biases.append((oc, t))
    else:
        units_in = layout.units_for(layer.c_i)
        units_out = layout.units_for(layer.c_o)
        swaps = (False, True) if layout.units > 1 and max(units_in, units_out) > 1 else (False,)
        for o in range(layout.ct_count(layer.c_o)):
            tl = []
            for b in range(len(in_cts)):
                for swap in swaps:
                    for d in range(1 - cpu, cpu):
                        for k, step in enumerate(taps):
                            bw = np.zeros((layout.units, cpu), dtype=np.int64)
                            for h in range(layout.units):
                                iu = layout.units * b + (h ^ int(swap))
                                ou = layout.units * o + h
                                if iu >= units_in or ou >= units_out:
                                    continue
                                for blk in range(max(0, -d), min(cpu, cpu - d)):
                                    ic, ocn = iu * cpu + blk + d, ou * cpu + blk
                                    if ic < layer.c_i and ocn < layer.c_o:
                                        bw[h, blk] = layer.weights[ocn, ic, k]
                            if not bw.any():
                                continue
                            tl.append((b, int((step + d * layout.tile) % layout.ring) % ring_slots, swap,
                                       pt_blocks(bw)))
            terms.append(tl)
    plan = cache[key] = {"terms": terms, "pt_rows": pt_rows, "biases": biases, "dev": {}}
    return plan


def conv_conventional(x: PackedTensor, layer: ConvLayerSpec, swks: bfv.SwitchingKeySet,
                      params: RingParams) -> PackedTensor:
    """Baseline: HRot per (tap, channel offset) + PMult by weight plaintexts
    + HAdd (conv.py:457-564). Same terms, same result; on the device the whole
    chain is one fused pass (fhe_rot_pmac: rotations key-switched in registers
    from hoisted digits, never written to HBM). FLASHHE_CONVENTIONAL=
    materialized selects the two-kernel form (batched K4 rotations + fhe_pmac)
    for A/B checks."""
    layout = x.layout
    if x.cts[0].encoding != Encoding.BATCH:
        raise EncodingError("conventional convolution needs batch-encoded input")
    if (layout.height, layout.width) != (layer.height, layer.width) or layout.pad != layer.f_w // 2:
        raise ParameterError("tensor layout does not match the layer geometry")
    in_cts = list(x.cts)
    for ct in in_cts:
        if ct.domain != Domain.EVAL:
            raise EncodingError("HRot operates in the evaluation domain")
    plan = _conventional_plan(layer, layout, len(in_cts), params)
    terms, pt_rows, biases = plan["terms"], plan["pt_rows"], plan["biases"]
    n = params.n
    needed = {(st, sw) for tl in terms for _, st, sw, _ in tl}
    for st, sw in needed:  # the reference raises KeyError for a missing key, EncodingError for a bad ct
        for ct in in_cts[:1]:
            if st:
                bfv._check_hrot(ct, st, swks)
            if sw:
                bfv._check_hrot(ct, bfv.COLUMN_ROTATION, swks)
    dev = device.require_cuda()
    n_out = len(terms)
    out = torch.empty((n_out, 2, n), dtype=torch.int64, device=dev)
    import os

    if needed and os.environ.get("FLASHHE_CONVENTIONAL", "fused") == "fused":
        _conventional_fused(in_cts, plan, swks, params, out)
    elif needed:
        R, index = _rotations(in_cts, needed, swks, params)
        pt = device.to_device(np.stack(pt_rows))
        pt_mont = torch.empty_like(pt)
        _native.call("fhe_to_montgomery", _native.u64_array([params.q]), 1, 1, len(pt_rows), n, pt.data_ptr(),
                     pt_mont.data_ptr(), device.stream())
        off = np.zeros(n_out + 1, dtype=np.int32)
        flat = []
        for o, tl in enumerate(terms):
            off[o + 1] = off[o] + len(tl)
            flat.extend((index[(b, st, sw)], p_) for b, st, sw, p_ in tl)
        tarr = np.asarray(flat, dtype=np.int32).reshape(-1, 2) if flat else np.zeros((1, 2), np.int32)
        assert tarr[:, 0].max(initial=0) < R.shape[0] and tarr[:, 1].max(initial=0) < len(pt_rows)
        ring._bump("modmul", 2 * n * len(flat))
        off_d = torch.from_numpy(off).to(dev)  # kept alive until the launch is enqueued
        terms_d = torch.from_numpy(np.ascontiguousarray(tarr)).to(dev)
        _native.call("fhe_pmac", params.q, n, R.data_ptr(), pt_mont.data_ptr(), off_d.data_ptr(), terms_d.data_ptr(),
                     n_out, out.data_ptr(), device.stream())
    else:
        out.zero_()
    out_cts = list(bfv.cts_from_rows(out, params.q, Encoding.BATCH, Domain.EVAL))
    if layout.fragmented:
        if layer.bias is not None:
            out_cts = [_conv_bias_batch(ct, layout, t, int(layer.bias[oc]), params) if layer.bias[oc] else ct
                       for ct, (oc, t) in zip(out_cts, biases)]
    elif layer.bias is not None and layer.bias.any():
        out_cts = _conv_bias_batch_packed(out_cts, layout, layer, params)
    return PackedTensor(out_cts, layout, layer.c_o, x.scale + layer.weight_scale)


def _conv_bias_batch(ct: Ciphertext, layout: TileLayout, pair: int, value: int, params: RingParams):
    vec = np.zeros(params.n, dtype=np.int64)
    tp = _interior(layout)
    for h in range(layout.units):
        k = pair * layout.units + h
        if k >= layout.frags:
            break
        sel = tp[tp // layout.frag_len == k]
        vec[h * layout.ring + layout.halo + sel - k * layout.frag_len] = value % params.p
    return bfv.plain_add(ct, bfv.encode_batch(vec, params), params)


def _conv_bias_batch_packed(out_cts, layout: TileLayout, layer: ConvLayerSpec, params: RingParams):
    tp = _interior(layout)
    fixed = []
    for o, ct in enumerate(out_cts):
        vec = np.zeros(params.n, dtype=np.int64)
        for h in range(layout.units):
            for blk in range(layout.c_n):
                oc = (layout.units * o + h) * layout.c_n + blk
                if oc >= layer.c_o:
                    break
                vec[h * layout.ring + blk * layout.tile + tp] = int(layer.bias[oc]) % params.p
        fixed.append(bfv.plain_add(ct, bfv.encode_batch(vec, params), params))
    return fixed


# ---------------------------------------------------------------------------
# storage accounting (conv.py:677-739), host-only


def conventional_plaintext_count(layer: ConvLayerSpec, params: RingParams) -> int:
    layout = layout_batch(params, layer.height, layer.width, layer.f_w)
    taps = layer.f_w * layer.f_w
    if layout.fragmented:
        return layer.c_o * layer.c_i * -(-layout.frags // layout.units) * taps
    return layout.ct_count(layer.c_o) * layout.ct_count(layer.c_i) * (2 * layout.c_n - 1) * taps


def storage_report(layers: list[ConvLayerSpec], params: RingParams, decomp_log: int = CONV_DECOMP_LOG) -> dict:
    """Server-side bytes of the two conv paths: raw int weights and no keys
    (proposed) vs weight plaintexts plus switching keys (conventional)."""
    digits = -(-params.q.bit_length() // decomp_log)
    steps = set()
    for layer in layers:
        steps.update(conventional_steps(layer, params))
    return {
        "proposed_weight_bytes": sum(l.c_o * l.c_i * l.f_w * l.f_w for l in layers),
        "proposed_swk_bytes": 0,
        "conventional_weight_bytes": sum(conventional_plaintext_count(l, params) for l in layers) * params.n * 8,
        "conventional_swk_bytes": len(steps) * digits * 2 * params.n * 8,
    }


VGG16_GEOMETRY = [
    (64, 64, 3, 64), (64, 64, 64, 64),
    (32, 32, 64, 128), (32, 32, 128, 128),
    (16, 16, 128, 256), (16, 16, 256, 256), (16, 16, 256, 256),
    (8, 8, 256, 512), (8, 8, 512, 512), (8, 8, 512, 512),
    (4, 4, 512, 512), (4, 4, 512, 512), (4, 4, 512, 512),
]


def vgg16_step_set(params: RingParams) -> list[int]:
    """Rotation steps of a conventional VGG-16 pipeline (unpadded row-major
    tiles, packed output channels) — the switching-key storage reference."""
    ring_slots = params.n // 2
    steps = set()
    for h, w, _, _ in VGG16_GEOMETRY:
        steps.update((dy * w + dx) % ring_slots for dy in (-1, 0, 1) for dx in (-1, 0, 1))
        if h * w <= ring_slots:
            steps.update(d * h * w % ring_slots for d in range(1, ring_slots // (h * w)))
    steps.discard(0)
    return sorted(steps)
