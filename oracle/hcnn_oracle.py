"""CPU ORACLE — test infrastructure only, never part of the product path.

A plain numpy / Python-int restatement of the reference (`hefir`, mounted at
/root/reference/pkg/src/hefir in the build container) for the homomorphic
evaluation hot path.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this module,
and only as the checker (or the timed CPU baseline), never as the thing that is
measured or shipped.

Pinning: `tests/test_oracle_pinned.py` checks every function here against the
golden vectors produced by the reference itself (`tests/golden/make_golden.py`,
which imports /root/reference through a `gmpy2 -> int` shim) and, when the
reference is importable, against the reference directly on fresh seeds.

Citations are `pkg/src/hefir/<file>:<line>` in /root/reference.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from math import prod

import numpy as np

# ---------------------------------------------------------------------------
# number theory (ntt.py:25-60)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (ntt.py:25-47)."""
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for sp in small:
        if n % sp == 0:
            return n == sp
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def primitive_2n_root(p: int, n: int) -> int:
    """First g^((p-1)/2N) (g = 2, 3, ...) whose N-th power is -1 (ntt.py:50-60).

    The reference's NTT domain is defined by exactly this root, so the search
    order matters for NTT-domain keys.
    """
    if (p - 1) % (2 * n):
        raise ValueError(f"{p} is not 1 mod {2 * n}")
    e = (p - 1) // (2 * n)
    g = 2
    while g < p:
        c = pow(g, e, p)
        if pow(c, n, p) == p - 1:
            return c
        g += 1
    raise ValueError("no primitive root")


def bitrev_perm(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    out = np.zeros(n, dtype=np.int64)
    for i in range(n):
        out[i] = int(format(i, f"0{bits}b")[::-1], 2) if bits else 0
    return out


# ---------------------------------------------------------------------------
# RNS context (ring.py:51-95)


class Context:
    """N, the RNS primes of q and their transform tables (ring.py:51-95)."""

    def __init__(self, n: int, primes):
        self.n = n
        self.primes = [int(p) for p in primes]
        self.k = len(self.primes)
        self.q = prod(self.primes)
        self.mods = np.array(self.primes, dtype=np.int64).reshape(-1, 1)
        self.psi = [primitive_2n_root(p, n) for p in self.primes]
        self.rev = bitrev_perm(n)
        jj = np.arange(n)
        self.twist = np.array(
            [[pow(s, int(j), p) for j in jj] for s, p in zip(self.psi, self.primes)],
            dtype=np.int64,
        )
        # inverse twist with N^-1 folded in (ntt.py:103-106)
        self.untwist = np.array(
            [
                [pow(s, -int(j), p) * pow(n, -1, p) % p for j in jj]
                for s, p in zip(self.psi, self.primes)
            ],
            dtype=np.int64,
        )
        # per-stage cyclic twiddles for a decimation-in-frequency transform
        self._dif_fwd = self._stage_tables(+1)
        self._dif_inv = self._stage_tables(-1)
        # CRT lift weights C_i = (q/p_i) * ((q/p_i)^-1 mod p_i)  (ring.py:73-77)
        self.crt_w = [
            (self.q // p) * pow((self.q // p) % p, -1, p) % self.q for p in self.primes
        ]
        h = hashlib.sha256()
        h.update(n.to_bytes(8, "little"))
        for p in self.primes:
            h.update(p.to_bytes(8, "little"))
        self.fingerprint = h.hexdigest()[:16]

    def _stage_tables(self, sign):
        tabs = []
        half = self.n // 2
        while half >= 1:
            rows = []
            for s, p in zip(self.psi, self.primes):
                w = pow(s * s % p, sign * (self.n // (2 * half)), p)
                rows.append([pow(w, j, p) for j in range(half)])
            tabs.append((half, np.array(rows, dtype=np.int64)))
            half //= 2
        return tabs

    def scalar_col(self, value: int) -> np.ndarray:
        return np.array([value % p for p in self.primes], dtype=np.int64).reshape(-1, 1)


def _cyclic_dif(a: np.ndarray, mods: np.ndarray, tabs) -> np.ndarray:
    """Cyclic NTT per row by Gentleman-Sande decimation in frequency.

    Output is bit-reversed; callers permute.  Same transform as the
    reference's bit-reverse + Cooley-Tukey (ntt.py:113-154), computed the other
    way round.
    """
    rows, n = a.shape
    a = a.copy()
    for half, tw in tabs:
        v = a.reshape(rows, n // (2 * half), 2, half)
        top = v[:, :, 0, :].copy()
        bot = v[:, :, 1, :].copy()
        m3 = mods.reshape(rows, 1, 1)
        v[:, :, 0, :] = (top + bot) % m3
        v[:, :, 1, :] = ((top - bot) % m3) * tw.reshape(rows, 1, half) % m3
    return a


def ntt_forward(ctx: Context, res: np.ndarray) -> np.ndarray:
    """Natural-order negacyclic NTT: out[k] = a(psi^(2k+1)) (ring.py:147-154)."""
    a = res * ctx.twist % ctx.mods
    out = _cyclic_dif(a, ctx.mods, ctx._dif_fwd)
    return out[:, ctx.rev]


def ntt_inverse(ctx: Context, res: np.ndarray) -> np.ndarray:
    """Inverse of ntt_forward (ring.py:156-163)."""
    a = _cyclic_dif(res, ctx.mods, ctx._dif_inv)[:, ctx.rev]
    return a * ctx.untwist % ctx.mods


def _wide_tables(p: int, n: int):
    psi = primitive_2n_root(p, n)
    fwd, inv = [], []
    half = n // 2
    while half >= 1:
        for sign, tabs in ((1, fwd), (-1, inv)):
            w = pow(psi * psi % p, sign * (n // (2 * half)), p)
            tabs.append((half, np.array([[pow(w, j, p) for j in range(half)]], dtype=object)))
        half //= 2
    twist = np.array([pow(psi, j, p) for j in range(n)], dtype=object)
    untwist = np.array([pow(psi, -j, p) * pow(n, -1, p) % p for j in range(n)], dtype=object)
    return fwd, inv, twist, untwist


def ntt_forward_wide(p: int, n: int, res) -> np.ndarray:
    """ntt_forward for one prime of up to 62 bits in Python ints (ring.py:45-46
    admits such primes; ring.py:147-154 / ntt.py:113-154 transform them):
    out[k] = a(psi^(2k+1)), natural order.  res: [rows][n] ints."""
    fwd, _, twist, _ = _wide_tables(p, n)
    mods = np.full((1, 1), p, dtype=object)
    rows = [np.array([[int(v) for v in r]], dtype=object) * twist % p for r in np.atleast_2d(res)]
    return np.concatenate([_cyclic_dif(a, mods, fwd)[:, bitrev_perm(n)] for a in rows])


def ntt_inverse_wide(p: int, n: int, res) -> np.ndarray:
    """Inverse of ntt_forward_wide (ring.py:156-163)."""
    _, inv, _, untwist = _wide_tables(p, n)
    mods = np.full((1, 1), p, dtype=object)
    rows = [np.array([[int(v) for v in r]], dtype=object) for r in np.atleast_2d(res)]
    return np.concatenate([_cyclic_dif(a, mods, inv)[:, bitrev_perm(n)] * untwist % p for a in rows])


# ---------------------------------------------------------------------------
# ring arithmetic (ring.py:170-207, 276-335)


def mul_scalar(ctx: Context, res: np.ndarray, w: int) -> np.ndarray:
    return res * ctx.scalar_col(int(w)) % ctx.mods


def crt_combine(residues, moduli) -> int:
    """Unique integer in [0, prod m) with the given residues (ring.py:276-283)."""
    total = prod(int(m) for m in moduli)
    acc = 0
    for r, m in zip(residues, moduli):
        big = total // int(m)
        acc += int(r) * big * pow(big % int(m), -1, int(m))
    return acc % total


def crt_lift(ctx: Context, res: np.ndarray) -> list:
    """Canonical [0, q) integers from residues (ring.py:286-295)."""
    acc = [0] * ctx.n
    for i in range(ctx.k):
        w = ctx.crt_w[i]
        row = res[i].tolist()
        acc = [a + int(r) * w for a, r in zip(acc, row)]
    return [a % ctx.q for a in acc]


def crt_reduce(ctx: Context, ints) -> np.ndarray:
    """Residue rows of integers (any sign) (ring.py:298-302)."""
    return np.array([[int(x) % p for x in ints] for p in ctx.primes], dtype=np.int64)


def negacyclic_exact(a, b, n: int, slot_bits: int) -> list:
    """Exact product in Z[X]/(X^N+1) of non-negative coefficient lists.

    Kronecker substitution with one big-integer multiply, as the reference
    does (ring.py:305-335); slots must not carry.
    """
    sb = (slot_bits + 7) // 8
    pa = int.from_bytes(b"".join(int(x).to_bytes(sb, "little") for x in a), "little")
    pb = int.from_bytes(b"".join(int(x).to_bytes(sb, "little") for x in b), "little")
    raw = (pa * pb).to_bytes(2 * n * sb, "little")
    lo = [int.from_bytes(raw[i * sb : (i + 1) * sb], "little") for i in range(n)]
    hi = [int.from_bytes(raw[(n + i) * sb : (n + i + 1) * sb], "little") for i in range(n)]
    return [x - y for x, y in zip(lo, hi)]


# ---------------------------------------------------------------------------
# BFV parameters and the multiplication path (bfv.py:45-91, 321-443)


class Params:
    """Plaintext modulus t, relin base w and derived constants (bfv.py:45-91)."""

    def __init__(self, ctx: Context, t: int, w: int = 1 << 16):
        self.ctx = ctx
        self.t = int(t)
        self.w = int(w)
        self.q_bits = ctx.q.bit_length()
        ell, acc = 0, self.w
        while acc <= ctx.q:
            acc *= self.w
            ell += 1
        self.l = ell
        self.delta = ctx.q // self.t
        self.slot_bits = 2 * self.q_bits + ctx.n.bit_length() + 1
        self.fingerprint = f"{ctx.fingerprint}:t{self.t}:w{self.w}"


def round_half_away_div(num: int, den: int) -> int:
    """round(num/den), ties away from zero (bfv.py:229-236, codec.py:18-24)."""
    if num >= 0:
        return (2 * num + den) // (2 * den)
    return -((-2 * num + den) // (2 * den))


def scale_round(pr: Params, d) -> np.ndarray:
    """round(t*d/q) mod q, back to residues (bfv.py:325-328)."""
    q = pr.ctx.q
    y = [round_half_away_div(int(x) * pr.t, q) % q for x in d]
    return crt_reduce(pr.ctx, y)


def tensor_square(pr: Params, c0: np.ndarray, c1: np.ndarray):
    """d0 = a0^2, d1 = 2 a0 a1, d2 = a1^2 over Z (bfv.py:331-338)."""
    n = pr.ctx.n
    a0 = crt_lift(pr.ctx, c0)
    a1 = crt_lift(pr.ctx, c1)
    d0 = negacyclic_exact(a0, a0, n, pr.slot_bits)
    x = negacyclic_exact(a0, a1, n, pr.slot_bits)
    d2 = negacyclic_exact(a1, a1, n, pr.slot_bits)
    return d0, [2 * v for v in x], d2


def tensor_mult(pr: Params, c, e):
    """General ct x ct tensor (bfv.py:339-347)."""
    n = pr.ctx.n
    a0, a1 = crt_lift(pr.ctx, c[0]), crt_lift(pr.ctx, c[1])
    b0, b1 = crt_lift(pr.ctx, e[0]), crt_lift(pr.ctx, e[1])
    d0 = negacyclic_exact(a0, b0, n, pr.slot_bits)
    x = negacyclic_exact(a0, b1, n, pr.slot_bits)
    y = negacyclic_exact(a1, b0, n, pr.slot_bits)
    d2 = negacyclic_exact(a1, b1, n, pr.slot_bits)
    return d0, [u + v for u, v in zip(x, y)], d2


def digits(pr: Params, c2: np.ndarray) -> np.ndarray:
    """Base-w digits of the canonical lift, shape (l+1, N) (bfv.py:350-365)."""
    vals = crt_lift(pr.ctx, c2)
    bits = pr.w.bit_length() - 1
    mask = pr.w - 1
    out = np.zeros((pr.l + 1, pr.ctx.n), dtype=np.int64)
    for j, v in enumerate(vals):
        for i in range(pr.l + 1):
            out[i, j] = (v >> (bits * i)) & mask
    return out


def relinearize(pr: Params, parts3, rlk_ntt) -> tuple:
    """Key switch of c2 with NTT-domain rlk [(k0_i, k1_i)] (bfv.py:368-404)."""
    ctx = pr.ctx
    c0, c1, c2 = parts3
    dg = digits(pr, c2)
    acc0 = np.zeros((ctx.k, ctx.n), dtype=np.int64)
    acc1 = np.zeros_like(acc0)
    for i in range(dg.shape[0]):
        rows = np.broadcast_to(dg[i], (ctx.k, ctx.n)) % ctx.mods
        dn = ntt_forward(ctx, rows)
        k0, k1 = rlk_ntt[i]
        acc0 = (acc0 + dn * k0 % ctx.mods) % ctx.mods
        acc1 = (acc1 + dn * k1 % ctx.mods) % ctx.mods
    out0 = (c0 + ntt_inverse(ctx, acc0)) % ctx.mods
    out1 = (c1 + ntt_inverse(ctx, acc1)) % ctx.mods
    return out0, out1


def hmult_raw(pr: Params, c, e=None) -> tuple:
    """3-part scaled tensor (bfv.py:407-416); e=None squares (bfv.py:441)."""
    if e is None:
        ds = tensor_square(pr, c[0], c[1])
    else:
        ds = tensor_mult(pr, c, e)
    return tuple(scale_round(pr, d) for d in ds)


def hsquare(pr: Params, c, rlk_ntt) -> tuple:
    """tensor -> scale -> relinearize (bfv.py:435-443)."""
    return relinearize(pr, hmult_raw(pr, c), rlk_ntt)


def hmult_plain(pr: Params, c, poly: np.ndarray) -> tuple:
    """Ciphertext times plaintext (bfv.py:301-318): the plaintext is lifted at
    its centred representative (bfv.py:110-112); a constant takes the scalar
    path (ring.py:193-196), anything else NTT(part) * NTT(lift) -> INTT."""
    ctx = pr.ctx
    t = pr.t
    poly = np.asarray(poly, dtype=np.int64)
    centered = np.where(poly > t // 2, poly - t, poly)
    if not centered[1:].any():
        return tuple(mul_scalar(ctx, part, int(centered[0])) for part in c)
    lifted = centered[None, :] % ctx.mods
    lf = ntt_forward(ctx, lifted)
    return tuple(ntt_inverse(ctx, ntt_forward(ctx, np.asarray(part, dtype=np.int64)) * lf % ctx.mods) for part in c)


# ---------------------------------------------------------------------------
# client side: keys, encryption, decryption (bfv.py:164-250), used only to
# cross-check the product's host client and to decrypt in tests


def _small_gauss(rng, n):
    out = np.rint(rng.normal(0.0, 3.2, n)).astype(np.int64)
    bad = np.abs(out) > 19
    while bad.any():
        out[bad] = np.rint(rng.normal(0.0, 3.2, int(bad.sum()))).astype(np.int64)
        bad = np.abs(out) > 19
    return out


def keygen(pr: Params, rng):
    """(s_bits, pk=(b_ntt, a_ntt), rlk=[(k0_ntt, k1_ntt)]) (bfv.py:164-188)."""
    ctx = pr.ctx
    s = rng.integers(0, 2, ctx.n, dtype=np.int64)
    s_ntt = ntt_forward(ctx, np.broadcast_to(s, (ctx.k, ctx.n)) % ctx.mods)
    s2_ntt = s_ntt * s_ntt % ctx.mods

    def uniform():
        return np.stack([rng.integers(0, p, ctx.n, dtype=np.int64) for p in ctx.primes])

    def noise_ntt():
        e = _small_gauss(rng, ctx.n)
        return ntt_forward(ctx, e[None, :] % ctx.mods)

    a = uniform()
    e = noise_ntt()
    b = (e - a * s_ntt % ctx.mods) % ctx.mods
    rlk = []
    wp = 1
    for _ in range(pr.l + 1):
        ai = uniform()
        ei = noise_ntt()
        k0 = (s2_ntt * ctx.scalar_col(wp) % ctx.mods - (ai * s_ntt % ctx.mods + ei)) % ctx.mods
        rlk.append((k0, ai))
        wp *= pr.w
    return s, (b, a), rlk


def encrypt(pr: Params, pk, m: np.ndarray, rng) -> tuple:
    """(c0, c1) of plaintext poly m in [0,t) (bfv.py:201-216)."""
    ctx = pr.ctx
    b, a = pk
    u = rng.integers(0, 2, ctx.n, dtype=np.int64)
    un = ntt_forward(ctx, np.broadcast_to(u, (ctx.k, ctx.n)) % ctx.mods)
    c0 = ntt_inverse(ctx, b * un % ctx.mods)
    c1 = ntt_inverse(ctx, a * un % ctx.mods)
    e1 = _small_gauss(rng, ctx.n)
    e2 = _small_gauss(rng, ctx.n)
    c0 = (c0 + e1[None, :]) % ctx.mods
    c1 = (c1 + e2[None, :]) % ctx.mods
    dm = ctx.scalar_col(pr.delta) * (np.asarray(m, dtype=np.int64)[None, :] % ctx.mods) % ctx.mods
    return ((c0 + dm) % ctx.mods, c1)


def decrypt(pr: Params, s_bits: np.ndarray, c) -> np.ndarray:
    """Exact-rounding decryption of a 2-part ct (bfv.py:219-250)."""
    ctx = pr.ctx
    s_ntt = ntt_forward(ctx, np.broadcast_to(s_bits, (ctx.k, ctx.n)) % ctx.mods)
    ph = (c[0] + ntt_inverse(ctx, ntt_forward(ctx, c[1]) * s_ntt % ctx.mods)) % ctx.mods
    v = crt_lift(ctx, ph)
    return np.array(
        [round_half_away_div(x * pr.t, ctx.q) % pr.t for x in v], dtype=np.int64
    )


# ---------------------------------------------------------------------------
# slot encoder over Z_t (batching.py:41-95)


class SlotCodec:
    """Slot i <-> evaluation at zeta^(2i+1) over Z_t (batching.py:41-95)."""

    def __init__(self, t: int, n: int):
        self.t, self.n = int(t), n
        z = primitive_2n_root(self.t, n)
        self.zeta = z
        self.points = [pow(z, 2 * i + 1, self.t) for i in range(n)]
        self.rev = bitrev_perm(n)
        t_ = self.t
        self.untwist = np.array(
            [pow(z, -j, t_) * pow(n, -1, t_) % t_ for j in range(n)], dtype=object
        )
        tabs = []
        half = n // 2
        while half >= 1:
            w = pow(z * z % t_, -(n // (2 * half)), t_)
            tabs.append((half, np.array([[pow(w, j, t_) for j in range(half)]], dtype=object)))
            half //= 2
        self._inv_tabs = tabs

    def encode(self, slots) -> np.ndarray:
        """Plaintext poly m with m(zeta^(2i+1)) = slots[i] (batching.py:78-87)."""
        a = np.array([[int(v) % self.t for v in slots]], dtype=object)
        mods = np.array([[self.t]], dtype=object)
        a = _cyclic_dif(a, mods, self._inv_tabs)[:, self.rev]
        return np.array([int(v) for v in (a[0] * self.untwist) % self.t], dtype=np.int64)

    def decode(self, m) -> np.ndarray:
        t = self.t
        out = []
        coeffs = [int(c) for c in m]
        for x in self.points:
            acc = 0
            for c in reversed(coeffs):
                acc = (acc * x + c) % t
            out.append(acc)
        return np.array(out, dtype=np.int64)


def pack_images(pr: Params, pk, codec: SlotCodec, images, rng) -> list:
    """One ct per pixel position, slot j = image j (engine.py:146-175)."""
    stack = np.stack([np.asarray(im, dtype=np.int64) for im in images])
    flat = stack.reshape(len(images), -1) % pr.t
    cts = []
    for pos in range(flat.shape[1]):
        slots = np.zeros(pr.ctx.n, dtype=np.int64)
        slots[: len(images)] = flat[:, pos]
        cts.append(encrypt(pr, pk, codec.encode(slots), rng))
    return cts


# ---------------------------------------------------------------------------
# the evaluator (engine.py:61-85, 206-423)


@dataclass
class Counter:
    """Same fields and semantics as engine.OpCounter (engine.py:61-85)."""

    mult_plain_scheduled: int = 0
    mult_plain_executed: int = 0
    mult_plain_skipped: int = 0
    hsquare: int = 0
    hadd: int = 0


@dataclass
class Tensor:
    shape: tuple  # (h, w, c)
    cts: list  # list of (c0, c1) residue arrays, (y, x, c) row-major
    delta: int = 1

    def at(self, y, x, ch):
        h, w, c = self.shape
        return self.cts[(y * w + x) * c + ch]


def weighted_sum(pr: Params, taps, counter: Counter):
    """sum w*ct, zero weights skipped but scheduled (engine.py:206-223)."""
    ctx = pr.ctx
    acc0 = acc1 = None
    used = 0
    for ct, w in taps:
        counter.mult_plain_scheduled += 1
        w = int(w)
        if w == 0:
            counter.mult_plain_skipped += 1
            continue
        counter.mult_plain_executed += 1
        used += 1
        t0 = mul_scalar(ctx, ct[0], w)
        t1 = mul_scalar(ctx, ct[1], w)
        acc0 = t0 if acc0 is None else (acc0 + t0) % ctx.mods
        acc1 = t1 if acc1 is None else (acc1 + t1) % ctx.mods
    if used == 0:
        z = np.zeros((ctx.k, ctx.n), dtype=np.int64)
        return (z, z.copy())
    counter.hadd += used - 1
    return (acc0, acc1)


def conv(pr, x: Tensor, kernel, stride, padded, groups, weight_scale, weights, counter) -> Tensor:
    """Grouped, strided, optionally padded conv (engine.py:237-303)."""
    h, w, c = x.shape
    f, kh, kw, cg = np.asarray(weights).shape
    sh, sw = stride
    ph = (kh - 1) // 2 if padded else 0
    pw = (kw - 1) // 2 if padded else 0
    oh = (h + 2 * ph - kh) // sh + 1
    ow = (w + 2 * pw - kw) // sw + 1
    per = f // groups
    out = []
    for oy in range(oh):
        for ox in range(ow):
            for fi in range(f):
                g = fi // per
                taps = []
                for ky in range(kh):
                    iy = oy * sh + ky - ph
                    if not 0 <= iy < h:
                        continue
                    for kx in range(kw):
                        ix = ox * sw + kx - pw
                        if not 0 <= ix < w:
                            continue
                        for ci in range(cg):
                            taps.append((x.at(iy, ix, g * cg + ci), weights[fi][ky][kx][ci]))
                out.append(weighted_sum(pr, taps, counter))
    return Tensor((oh, ow, f), out, x.delta * weight_scale)


def fc(pr, x: Tensor, weights, weight_scale, counter) -> Tensor:
    """out[o] = sum_i W[o, i] flat[i] (engine.py:306-334)."""
    weights = np.asarray(weights)
    out = [weighted_sum(pr, list(zip(x.cts, weights[o])), counter) for o in range(weights.shape[0])]
    return Tensor((1, 1, weights.shape[0]), out, x.delta * weight_scale)


def pool(pr, x: Tensor, extent, stride, counter) -> Tensor:
    """Window sum via hadd chain (engine.py:367-397)."""
    ctx = pr.ctx
    h, w, c = x.shape
    sh, sw = stride
    oh = (h - extent) // sh + 1
    ow = (w - extent) // sw + 1
    out = []
    for oy in range(oh):
        for ox in range(ow):
            for ch in range(c):
                acc = None
                for dy in range(extent):
                    for dx in range(extent):
                        ct = x.at(oy * sh + dy, ox * sw + dx, ch)
                        if acc is None:
                            acc = ct
                        else:
                            acc = ((acc[0] + ct[0]) % ctx.mods, (acc[1] + ct[1]) % ctx.mods)
                            counter.hadd += 1
                out.append(acc)
    return Tensor((oh, ow, c), out, x.delta * extent * extent)


def square(pr, x: Tensor, rlk_ntt, counter) -> Tensor:
    """hsquare on every ciphertext (engine.py:337-364)."""
    out = [hsquare(pr, ct, rlk_ntt) for ct in x.cts]
    counter.hsquare += len(out)
    return Tensor(x.shape, out, x.delta * x.delta)


def plain_forward(layers, image):
    """Plaintext integer network (nn_oracle.py:230-311): conv, square, pool, fc
    on exact Python ints; `layers` as for `network`."""
    x = np.asarray(image, dtype=object)
    for L in layers:
        k = L["kind"]
        if k == "conv":
            w = np.asarray(L["weights"], dtype=object)
            f, kh, kw, cg = w.shape
            h, wd, c = x.shape
            sh, sw = L["stride"]
            ph = (kh - 1) // 2 if L["padded"] else 0
            pw = (kw - 1) // 2 if L["padded"] else 0
            xp = np.zeros((h + 2 * ph, wd + 2 * pw, c), dtype=object)
            xp[ph:ph + h, pw:pw + wd] = x
            oh = (h + 2 * ph - kh) // sh + 1
            ow = (wd + 2 * pw - kw) // sw + 1
            per = f // L["groups"]
            out = np.zeros((oh, ow, f), dtype=object)
            for oy in range(oh):
                for ox in range(ow):
                    win = xp[oy * sh:oy * sh + kh, ox * sw:ox * sw + kw]
                    for fi in range(f):
                        g = fi // per
                        out[oy, ox, fi] = int((win[:, :, g * cg:(g + 1) * cg] * w[fi]).sum())
            x = out
        elif k == "square":
            x = x * x
        elif k == "pool":
            e = L["extent"]
            sh, sw = L["stride"]
            h, wd, c = x.shape
            oh, ow = (h - e) // sh + 1, (wd - e) // sw + 1
            out = np.zeros((oh, ow, c), dtype=object)
            for oy in range(oh):
                for ox in range(ow):
                    out[oy, ox] = x[oy * sh:oy * sh + e, ox * sw:ox * sw + e].sum(axis=(0, 1))
            x = out
        elif k == "fc":
            w = np.asarray(L["weights"], dtype=object)
            x = (w @ x.reshape(-1)).reshape(1, 1, -1)
    return x


def network(pr, x: Tensor, layers, rlk_ntt, counter=None, hook=None) -> Tensor:
    """Layer loop (engine.py:400-423).

    `layers` is a list of dicts: {"kind": "conv"|"square"|"pool"|"fc", ...}.
    """
    counter = counter if counter is not None else Counter()
    for L in layers:
        k = L["kind"]
        if k == "conv":
            x = conv(pr, x, L["kernel"], L["stride"], L["padded"], L["groups"],
                     L["weight_scale"], L["weights"], counter)
        elif k == "square":
            x = square(pr, x, rlk_ntt, counter)
        elif k == "pool":
            x = pool(pr, x, L["extent"], L["stride"], counter)
        elif k == "fc":
            x = fc(pr, x, L["weights"], L["weight_scale"], counter)
        if hook is not None:
            hook(L["name"], x)
    return x


# ---------------------------------------------------------------------------
# digests used by the golden fixtures


def tensor_digest(cts) -> str:
    """sha256 over u64-LE residues of a list of (c0, c1) in order."""
    h = hashlib.sha256()
    for ct in cts:
        for part in ct:
            h.update(np.ascontiguousarray(np.asarray(part, dtype="<u8")).tobytes())
    return h.hexdigest()
