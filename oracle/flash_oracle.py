"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain numpy / Python-int restatement of the reference algorithms on the hot
path (privinfer, /root/reference/pkg/src/privinfer). Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s CPU-baseline legs may import it,
and only as the checker (or the timed CPU baseline) — never as a product
path. Every function cites the reference lines it follows.

Pinned: tests/test_oracle_golden.py checks each function against golden
vectors produced by the reference itself (tests/golden/make_golden.py).

Exactness: all modular results are canonical [0, q) Python-int residues of
exact integer sums, as in the reference's object-array arithmetic.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------- NTT plan


def bitrev(x: int, bits: int) -> int:
    r = 0
    for _ in range(bits):
        r = (r << 1) | (x & 1)
        x >>= 1
    return r


def find_root(n: int, q: int) -> int:
    """ring.NttPlan._find_root (ring.py:121-127)."""
    e = (q - 1) // (2 * n)
    for g in range(2, 10000):
        psi = pow(g, e, q)
        if pow(psi, n, q) == q - 1:
            return psi
    raise ValueError("no 2n-th root of unity")


def ntt_tables(n: int, q: int):
    """psi_brv, ipsi_brv, n_inv (ring.py:96-113) as Python-int lists."""
    bits = n.bit_length() - 1
    psi = find_root(n, q)
    ipsi = pow(psi, -1, q)
    psi_brv = [pow(psi, bitrev(i, bits), q) for i in range(n)]
    ipsi_brv = [pow(ipsi, bitrev(i, bits), q) for i in range(n)]
    return psi_brv, ipsi_brv, pow(n, -1, q)


_tables: dict = {}


def _tab(n, q):
    if (n, q) not in _tables:
        _tables[(n, q)] = ntt_tables(n, q)
    return _tables[(n, q)]


def ntt_fwd(a, q: int) -> np.ndarray:
    """Cooley-Tukey, merged twiddles psi_brv[m+i], bit-reversed output
    (ring.py:129-144), on object (big-int) arrays."""
    a = np.array([int(v) for v in np.asarray(a).ravel()], dtype=object)
    n = len(a)
    psi_brv = np.array(_tab(n, q)[0], dtype=object)
    m, t = 1, n
    while m < n:
        t //= 2
        blk = a.reshape(m, 2 * t)
        u = blk[:, :t].copy()
        v = (blk[:, t:] * psi_brv[m : 2 * m, None]) % q
        blk[:, :t] = (u + v) % q
        blk[:, t:] = (u - v) % q
        m *= 2
    return a.astype(np.int64)


def ntt_inv(a, q: int) -> np.ndarray:
    """Gentleman-Sande with ipsi_brv[h+i], then × n^-1 (ring.py:146-162)."""
    a = np.array([int(v) for v in np.asarray(a).ravel()], dtype=object)
    n = len(a)
    _, ipsi_brv, n_inv = _tab(n, q)
    ipsi_brv = np.array(ipsi_brv, dtype=object)
    t, m = 1, n
    while m > 1:
        h = m // 2
        blk = a.reshape(h, 2 * t)
        u = blk[:, :t].copy()
        w = blk[:, t:].copy()
        blk[:, :t] = (u + w) % q
        blk[:, t:] = ((u - w) * ipsi_brv[h : 2 * h, None]) % q
        t *= 2
        m //= 2
    return ((a * n_inv) % q).astype(np.int64)


def pointwise(a, b, q: int) -> np.ndarray:
    """NttPlan.pointwise (ring.py:193-197)."""
    return ((np.asarray(a).astype(object) * np.asarray(b).astype(object)) % q).astype(np.int64)


def eval_perm(n: int, gpow: int) -> np.ndarray:
    """NttPlan.eval_perm (ring.py:199-202)."""
    bits = n.bit_length() - 1
    exp_at = np.array([2 * bitrev(i, bits) + 1 for i in range(n)], dtype=np.int64)
    index_of = np.full(2 * n, -1, dtype=np.int64)
    index_of[exp_at] = np.arange(n)
    return index_of[exp_at * gpow % (2 * n)]


# --------------------------------------------------------- coefficient ops


def monomial_mul(a, shift: int, q: int) -> np.ndarray:
    """a·x^(−shift) mod x^n+1 (ring.py:279-299)."""
    a = np.asarray(a, dtype=np.int64)
    n = len(a)
    s = shift % (2 * n)
    flip = s >= n
    s -= n if flip else 0
    rolled = np.concatenate([a[s:], a[:s]])
    wrapped = np.zeros(n, dtype=bool)
    wrapped[n - s :] = True
    neg = wrapped ^ flip
    return np.where(neg & (rolled != 0), q - rolled, rolled)


def apply_galois(a, gpow: int, q: int) -> np.ndarray:
    """a(x^gpow) with negacyclic signs (ring.py:326-334)."""
    a = np.asarray(a, dtype=np.int64)
    n = len(a)
    e = np.arange(n, dtype=np.int64) * gpow % (2 * n)
    out = np.empty(n, dtype=np.int64)
    out[e % n] = np.where((e >= n) & (a != 0), q - a, a)
    return out


def negacyclic_schoolbook(f, g, q: int) -> np.ndarray:
    """O(n²) negacyclic product (SPEC.md:57-63 oracle)."""
    f = [int(v) for v in f]
    g = [int(v) for v in g]
    n = len(f)
    out = [0] * n
    for i, fi in enumerate(f):
        if not fi:
            continue
        for j, gj in enumerate(g):
            k = i + j
            if k < n:
                out[k] += fi * gj
            else:
                out[k - n] -= fi * gj
    return np.array([v % q for v in out], dtype=np.int64)


# --------------------------------------------------------- Flash conv core


def _ext(a: np.ndarray, q: int) -> np.ndarray:
    """[−a | a | −a] with −a represented as q − a (conv._ExtPoly, conv.py:251-266)."""
    neg = np.where(a == 0, 0, q - a)
    return np.concatenate([neg, a, neg])


def lazy_sum(rows: np.ndarray, weights: np.ndarray, q: int) -> np.ndarray:
    """Σ_k w_k·rows_k mod q via two 30-bit limbs (WidePoly, ring.py:374-406).
    rows: int64 [K, n] in [0, q); weights: int [K]."""
    w = np.asarray(weights, dtype=np.int64)
    lo = (rows & ((1 << 30) - 1)).T @ w
    hi = (rows >> 30).T @ w
    return np.array([((int(h) << 30) + int(l)) % q for l, h in zip(lo, hi)], dtype=np.int64)


def conv_proposed(cts: np.ndarray, weights: np.ndarray, layout: dict, q: int,
                  channels=None) -> np.ndarray:
    """conv.conv_proposed / _proposed_channel (conv.py:326-411).

    cts: int64 [n_in, 2, n]; weights [c_o, c_i, f_w²]; layout dict with keys
    n, w_p, pad, tile, c_n, frags (TileLayout fields). Returns
    [len(channels)·frags, 2, n] in output order i·frags + k.
    For each output channel i and fragment k: partial = Σ_j DRot(t_j, tile·(j mod c_n)),
    t_j = Σ_taps w·DRot(ct_src, step) — the closed form of both DRots
    (x^(−a)·x^(−b) = x^(−(a+b))) is applied per term.
    """
    n = layout["n"]
    c_o, c_i, taps = weights.shape
    f_w = int(round(taps ** 0.5))
    pad = f_w // 2
    dy, dx = np.mgrid[0:f_w, 0:f_w]
    steps = ((dy - pad) * layout["w_p"] + (dx - pad)).ravel()          # conv.py:245-248
    frags = layout["frags"]
    exts = [[_ext(ct[p], q) for p in range(2)] for ct in cts]
    chans = range(c_o) if channels is None else channels
    out = np.zeros((len(chans) * frags, 2, n), dtype=np.int64)
    for oi, i in enumerate(chans):
        for k in range(frags):
            rows, wts = [[], []], []
            for j in range(c_i):
                src = j * frags + k if frags > 1 else j // layout["c_n"]
                shift = 0 if frags > 1 else layout["tile"] * (j % layout["c_n"])
                for t in range(taps):
                    w = int(weights[i, j, t])
                    if w == 0:
                        continue
                    total = int(steps[t]) + shift     # DRot(DRot(ct, step), shift)
                    wts.append(w)
                    for p in range(2):
                        if -n < total < n:
                            rows[p].append(exts[src][p][n + total : 2 * n + total])
                        else:
                            rows[p].append(monomial_mul(cts[src][p], total, q))
            for p in range(2):
                if wts:
                    out[oi * frags + k, p] = lazy_sum(np.stack(rows[p]), np.array(wts), q)
    return out


def add_bias(out: np.ndarray, bias_vals, masks: np.ndarray, delta: int, p: int, q: int) -> np.ndarray:
    """bfv.plain_add of the per-channel bias plaintexts (conv.py:408-424)."""
    out = out.copy()
    frags = masks.shape[0]
    for u in range(out.shape[0]):
        b = int(bias_vals[u // frags])
        if b:
            dm = delta * (b % p) * masks[u % frags].astype(np.int64)
            c0 = out[u, 0] + dm
            out[u, 0] = c0 - (c0 >= q) * q
    return out


def bias_masks(lay: dict) -> np.ndarray:
    """Slots of conv._bias_plaintext (conv.py:414-424), one row per fragment."""
    ys = lay["pad"] + np.arange(lay["height"])
    xs = lay["pad"] + np.arange(lay["width"])
    tp = (ys[:, None] * lay["w_p"] + xs[None, :]).ravel()
    masks = np.zeros((lay["frags"], lay["n"]), dtype=np.uint8)
    for f in range(lay["frags"]):
        if lay["frags"] > 1:
            sel = tp[tp // lay["frag_len"] == f]
            masks[f, lay["halo"] + sel - f * lay["frag_len"]] = 1
        else:
            masks[f, tp] = 1
    return masks


def avg_pool(cts: np.ndarray, k: int, w_p: int, q: int) -> np.ndarray:
    """conv.avg_pool (conv.py:604-623): Σ_{dy,dx<k} DRot(ct, dy·W_p+dx)."""
    n = cts.shape[-1]
    steps = [dy * w_p + dx for dy in range(k) for dx in range(k)]
    out = np.zeros_like(cts)
    for c, ct in enumerate(cts):
        for p in range(2):
            e = _ext(ct[p], q)
            out[c, p] = lazy_sum(np.stack([e[n + s : 2 * n + s] for s in steps]), np.ones(len(steps)), q)
    return out


def fully_connected(cts: np.ndarray, weights: np.ndarray, ct_idx, slots, q: int) -> np.ndarray:
    """conv.fully_connected (conv.py:626-668): row o = Σ_v W[o,v]·DRot(ct(v), slot(v))."""
    n = cts.shape[-1]
    exts = [[_ext(ct[p], q) for p in range(2)] for ct in cts]
    out = np.zeros((weights.shape[0], 2, n), dtype=np.int64)
    for o in range(weights.shape[0]):
        nz = [v for v in range(weights.shape[1]) if weights[o, v]]
        for p in range(2):
            if nz:
                rows = np.stack([exts[ct_idx[v]][p][n + slots[v] : 2 * n + slots[v]] for v in nz])
                out[o, p] = lazy_sum(rows, weights[o, nz], q)
    return out


# ----------------------------------------------------- BFV ops (bfv.py)


def hrot(c0, c1, gpow: int, keys, T: int, q: int):
    """bfv.hrot (bfv.py:467-500): keys = list of (swk0, swk1) EVAL arrays."""
    n = len(c0)
    perm = eval_perm(n, gpow)
    c1_coeff = ntt_inv(c1, q)
    acc0 = np.asarray(c0, dtype=np.int64)[perm].astype(object)
    acc1 = np.zeros(n, dtype=object)
    mask = (1 << T) - 1
    for i, (k0, k1) in enumerate(keys):
        d = ntt_fwd((c1_coeff >> (T * i)) & mask, q)[perm].astype(object)
        acc0 = acc0 + d * np.asarray(k0).astype(object)
        acc1 = acc1 + d * np.asarray(k1).astype(object)
    return (acc0 % q).astype(np.int64), (acc1 % q).astype(np.int64)


def galois_element(step: int, n: int) -> int:
    """bfv._galois_element (bfv.py:461-464); −1 selects the orbit swap."""
    return 2 * n - 1 if step == -1 else pow(3, int(step), 2 * n)


def decrypt_phase(c0, c1, s, q: int, eval_domain: bool = False) -> np.ndarray:
    """bfv._raw_phase (bfv.py:266-275) with s in the coefficient domain."""
    s_eval = ntt_fwd(s, q)
    if eval_domain:
        return ntt_inv((pointwise(c1, s_eval, q).astype(object) + np.asarray(c0).astype(object)) % q, q)
    c1s = ntt_inv(pointwise(ntt_fwd(c1, q), s_eval, q), q)
    return ((c1s.astype(object) + np.asarray(c0).astype(object)) % q).astype(np.int64)


def decrypt_round(u, q: int, p: int):
    """bfv.decrypt_with_budget rounding (bfv.py:285-293): (m, max|w|)."""
    delta = q // p
    u = np.asarray(u).astype(object)
    m_raw = (u + delta // 2) // delta
    w = u - delta * m_raw
    return (m_raw % p).astype(np.int64), int(max(abs(int(x)) for x in w))


def add_delta(base, m, q: int, p: int) -> np.ndarray:
    """c0 + Δ·(m mod p), one conditional subtract (bfv.py:248-263, 330-340)."""
    delta = q // p
    c = np.asarray(base, dtype=np.int64) + delta * (np.asarray(m, dtype=np.int64) % p)
    return c - (c >= q) * q


def x2x_client(w, p: int, f: int = 0) -> np.ndarray:
    """(w² + w·2^f) mod p."""
    w = np.asarray(w).astype(object)
    return ((w * w + w * (1 << f)) % p).astype(np.int64)


def x2x_server_const(r, r_sq, v, p: int, f: int = 0) -> np.ndarray:
    """(r² − r·2^f + v) mod p."""
    r = np.asarray(r).astype(object)
    return ((np.asarray(r_sq).astype(object) - r * (1 << f) + np.asarray(v).astype(object)) % p).astype(np.int64)


# ------------------------------------------- host sampling (bfv.py:64-90)
# Same numpy Generator calls in the same order as the reference, so a seeded
# rng reproduces its keys / encryptions exactly.


def sample_uniform(n: int, q: int, rng) -> np.ndarray:
    return rng.integers(0, q, n, dtype=np.int64)


def sample_error(n: int, cbd_k: int, rng) -> np.ndarray:
    bits = rng.integers(0, 2, (n, 2 * cbd_k), dtype=np.int64)
    return bits[:, :cbd_k].sum(axis=1) - bits[:, cbd_k:].sum(axis=1)


def keygen(n: int, q: int, rng) -> np.ndarray:
    """bfv.keygen (bfv.py:77-82): ternary s stored mod q."""
    t = rng.integers(-1, 2, n, dtype=np.int64)
    return np.where(t < 0, q - 1, t)


def expand_seed(seed: bytes, n: int, q: int) -> np.ndarray:
    """bfv.expand_seed (bfv.py:85-90)."""
    import hashlib

    key = int.from_bytes(hashlib.sha256(seed).digest()[:16], "little")
    return np.random.Generator(np.random.Philox(key=key)).integers(0, q, n, dtype=np.int64)


def encrypt_private(m, s, n: int, q: int, p: int, cbd_k: int, rng):
    """bfv.encrypt_private (bfv.py:171-189) -> (c0, c1, seed)."""
    seed = rng.bytes(32)
    a = expand_seed(seed, n, q)
    a_s = ntt_inv(pointwise(ntt_fwd(a, q), ntt_fwd(s, q), q), q)
    e = sample_error(n, cbd_k, rng)
    delta = q // p
    c0 = ((delta * (np.asarray(m, dtype=np.int64) % p)).astype(object) - a_s.astype(object) - e.astype(object)) % q
    return c0.astype(np.int64), a, seed


def gen_switching_keys(s, steps, n: int, q: int, cbd_k: int, T: int, rng) -> dict:
    """bfv.gen_switching_keys (bfv.py:431-458): {step: [(swk0, swk1)]*l}."""
    l = -(-q.bit_length() // T)
    s_eval = ntt_fwd(s, q).astype(object)
    keys = {}
    for step in steps:
        s_rot_eval = ntt_fwd(apply_galois(s, galois_element(step, n), q), q).astype(object)
        digits = []
        for i in range(l):
            a_eval = sample_uniform(n, q, rng)
            e_eval = ntt_fwd(sample_error(n, cbd_k, rng) % q, q).astype(object)
            target = s_rot_eval * pow(2, T * i, q) % q
            swk0 = (-(a_eval.astype(object) * s_eval % q + e_eval) + target) % q
            digits.append((swk0.astype(np.int64), a_eval))
        keys[int(step)] = digits
    return keys
