"""Host-side BFV types and the client operations (key generation, encryption,
decryption, slot encoding), mirroring the reference's data model.

The GPU evaluator (engine.py) accepts the reference's own objects (hefir
RnsContext / BfvParams / Ciphertext / RelinKey) or these mirrors — they expose
the same attributes.  These mirrors exist because the GPU box has no
reference tree; keygen/encrypt reproduce the reference's RNG draw order so the
same seed yields the same bytes (pinned in tests/test_client.py).

This is client code (it holds or uses the secret key); it is not on the
homomorphic-evaluation hot path, which runs only on the GPU.

Reference: ring.py:31-112 (RnsContext, RingElem), bfv.py:45-250 (params,
keys, encrypt, decrypt), batching.py:21-95 (slot encoder).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass
from enum import Enum
from math import prod

import numpy as np

from .errors import EncodingError, ParameterMismatchError, UnsupportedParametersError

NOISE_SIGMA = 3.2
NOISE_BOUND = 19


class Domain(Enum):
    COEFF = "coefficient"
    NTT = "ntt"


# ---------------------------------------------------------------- number theory


def is_prime(n: int) -> bool:
    if n < 2:
        return False
    bases = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for b in bases:
        if n % b == 0:
            return n == b
    d, r = n - 1, 0
    while not d & 1:
        d >>= 1
        r += 1
    for a in bases:
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


def primitive_root_2n(p: int, n: int) -> int:
    """The reference's psi: first g^((p-1)/2N), g = 2, 3, ... with psi^N = -1
    (ntt.py:50-60)."""
    if (p - 1) % (2 * n):
        raise ValueError(f"{p} is not 1 mod {2 * n}")
    e = (p - 1) // (2 * n)
    for g in range(2, p):
        c = pow(g, e, p)
        if pow(c, n, p) == p - 1:
            return c
    raise ValueError("no primitive root")


def _bitrev(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    idx = np.arange(n)
    out = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        out |= ((idx >> b) & 1) << (bits - 1 - b)
    return out


def _mulmod_split(a, b, m, chunks: int):
    """a * b mod m for int64 arrays with a, b < m < 2^47: a is consumed in
    15-bit chunks so every partial product stays below 2^63."""
    r = None
    for c in range(chunks - 1, -1, -1):
        part = (a >> (15 * c)) & 0x7FFF
        r = part * b % m if r is None else ((r << 15) + part * b) % m
    return r


class _Transform:
    """Natural-order negacyclic NTT over one modulus per row (numpy), the
    reference's NTT-domain convention: out[k] = a(psi^(2k+1)).

    int64 products for moduli < 2^31; moduli < 2^47 (e.g. the 43-bit MNIST
    plaintext modulus) use a chunked int64 multiply; larger ones Python ints.
    """

    def __init__(self, n: int, mods, psis, obj: bool = False):
        self.n = n
        top = max(int(m) for m in mods)
        self.split = 0
        if top >= (1 << 31) and top < (1 << 47):
            self.split = (top.bit_length() + 14) // 15
            obj = False
        self.obj = obj
        dt = object if obj else np.int64
        self.mods = np.array([int(m) for m in mods], dtype=dt).reshape(-1, 1)
        self.rev = _bitrev(n)
        j = list(range(n))
        self.twist = np.array([[pow(s, i, m) for i in j] for s, m in zip(psis, mods)], dtype=dt)
        self.untwist = np.array(
            [[pow(s, -i, m) * pow(n, -1, m) % m for i in j] for s, m in zip(psis, mods)], dtype=dt
        )
        self.fwd = self._tables(psis, mods, 1, dt)
        self.inv = self._tables(psis, mods, -1, dt)

    def _tables(self, psis, mods, sign, dt):
        out = []
        half = self.n // 2
        while half:
            rows = []
            for s, m in zip(psis, mods):
                w = pow(s * s % m, sign * (self.n // (2 * half)), m)
                rows.append([pow(w, i, m) for i in range(half)])
            out.append((half, np.array(rows, dtype=dt)))
            half //= 2
        return out

    def _mul(self, a, b, m):
        if self.split:
            return _mulmod_split(a, b, m, self.split)
        return a * b % m

    def _dif(self, a, tabs, mods):
        rows = a.shape[0]
        a = a.copy()
        m3 = mods.reshape(rows, 1, 1)
        for half, tw in tabs:
            v = a.reshape(rows, self.n // (2 * half), 2, half)
            u = v[:, :, 0, :].copy()
            w = v[:, :, 1, :].copy()
            v[:, :, 0, :] = (u + w) % m3
            v[:, :, 1, :] = self._mul((u - w) % m3, tw.reshape(rows, 1, half), m3)
        return a[:, self.rev]

    def forward(self, a, sel=None):
        mods = self.mods if sel is None else self.mods[sel]
        tw = self.twist if sel is None else self.twist[sel]
        tabs = self.fwd if sel is None else [(h, t[sel]) for h, t in self.fwd]
        return self._dif(self._mul(a % mods, tw, mods), tabs, mods)

    def inverse(self, a, sel=None):
        mods = self.mods if sel is None else self.mods[sel]
        ut = self.untwist if sel is None else self.untwist[sel]
        tabs = self.inv if sel is None else [(h, t[sel]) for h, t in self.inv]
        return self._mul(self._dif(a, tabs, mods), ut, mods)


# ---------------------------------------------------------------- ring


@dataclass(frozen=True)
class PrimeModulus:
    value: int
    n_root: int


class RnsContext:
    """N and the RNS primes of q (ring.py:51-95)."""

    def __init__(self, ring_degree: int, primes):
        if ring_degree < 4 or ring_degree & (ring_degree - 1):
            raise ValueError("ring degree must be a power of two >= 4")
        primes = [int(p) for p in primes]
        if len(set(primes)) != len(primes):
            raise ValueError("primes must be pairwise distinct")
        for p in primes:
            if not is_prime(p):
                raise ValueError(f"{p} is not prime")
            if p % (2 * ring_degree) != 1:
                raise ValueError(f"{p} is not 1 mod 2N")
        self.ring_degree = ring_degree
        psis = [primitive_root_2n(p, ring_degree) for p in primes]
        self.primes = tuple(PrimeModulus(p, s) for p, s in zip(primes, psis))
        self.prime_values = np.array(primes, dtype=np.int64)
        self.q_big = prod(primes)
        self._modcol = self.prime_values.reshape(-1, 1)
        self._ntt = None
        h = hashlib.sha256()
        h.update(ring_degree.to_bytes(8, "little"))
        for p in primes:
            h.update(p.to_bytes(8, "little"))
        self.fingerprint = h.hexdigest()[:16]

    @property
    def ntt(self) -> _Transform:
        if self._ntt is None:
            self._ntt = _Transform(self.ring_degree, [p.value for p in self.primes],
                                   [p.n_root for p in self.primes])
        return self._ntt

    def reduce_scalar(self, value: int) -> np.ndarray:
        return np.array([int(value) % p.value for p in self.primes], dtype=np.int64).reshape(-1, 1)

    def __eq__(self, other):
        return hasattr(other, "fingerprint") and self.fingerprint == other.fingerprint

    def __hash__(self):
        return hash(self.fingerprint)


class RingElem:
    __slots__ = ("ctx", "residues", "domain")

    def __init__(self, ctx, residues: np.ndarray, domain: Domain):
        self.ctx = ctx
        self.residues = residues
        self.domain = domain


def ntt_forward(e: RingElem) -> RingElem:
    return RingElem(e.ctx, e.ctx.ntt.forward(e.residues), Domain.NTT)


def ntt_inverse(e: RingElem) -> RingElem:
    return RingElem(e.ctx, e.ctx.ntt.inverse(e.residues), Domain.COEFF)


def zero_elem(ctx, domain: Domain = Domain.COEFF) -> RingElem:
    return RingElem(ctx, np.zeros((len(ctx.primes), ctx.ring_degree), dtype=np.int64), domain)


# ---------------------------------------------------------------- BFV


class BfvParams:
    """Plaintext modulus, relin base and derived constants (bfv.py:45-91)."""

    def __init__(self, ctx: RnsContext, plaintext_modulus: int, relin_base: int = 1 << 16,
                 depth: int = 0, security_bits: int = 0):
        if plaintext_modulus < 2:
            raise ParameterMismatchError("plaintext modulus must be >= 2")
        if plaintext_modulus >= ctx.q_big:
            raise ParameterMismatchError("plaintext modulus must be below q")
        if relin_base not in (1 << 8, 1 << 16, 1 << 32):
            raise ParameterMismatchError("relin base must be 2^8, 2^16 or 2^32")
        self.ctx = ctx
        self.t = int(plaintext_modulus)
        self.w = int(relin_base)
        self.depth = depth
        self.security_bits = security_bits
        q = ctx.q_big
        self.q_bits = q.bit_length()
        ell, acc = 0, self.w
        while acc <= q:
            acc *= self.w
            ell += 1
        self.l = ell
        self.delta = q // self.t
        self.delta_col = ctx.reduce_scalar(self.delta)
        self.tensor_slot_bits = 2 * self.q_bits + ctx.ring_degree.bit_length() + 1
        self.fingerprint = f"{ctx.fingerprint}:t{self.t}:w{self.w}"

    @property
    def ring_degree(self) -> int:
        return self.ctx.ring_degree

    def __eq__(self, other):
        return hasattr(other, "fingerprint") and self.fingerprint == other.fingerprint

    def __hash__(self):
        return hash(self.fingerprint)


@dataclass
class Plaintext:
    """Polynomial with coefficients in [0, t) (bfv.py:95-112)."""

    poly: np.ndarray
    t: int

    def __post_init__(self):
        self.poly = np.asarray(self.poly, dtype=np.int64)

    @staticmethod
    def constant(value: int, params) -> "Plaintext":
        poly = np.zeros(params.ring_degree, dtype=np.int64)
        poly[0] = value % params.t
        return Plaintext(poly, params.t)

    def centered(self) -> np.ndarray:
        half = self.t // 2
        return np.where(self.poly > half, self.poly - self.t, self.poly)


@dataclass
class SecretKey:
    s_bits: np.ndarray
    s_ntt: RingElem
    s2_ntt: RingElem


@dataclass
class PublicKey:
    b_ntt: RingElem
    a_ntt: RingElem
    fingerprint: str


@dataclass
class RelinKey:
    components: list
    base: int
    fingerprint: str


@dataclass
class Ciphertext:
    parts: tuple
    fingerprint: str
    is_fresh: bool = False

    def __len__(self):
        return len(self.parts)


def _gauss(rng, n):
    out = np.rint(rng.normal(0.0, NOISE_SIGMA, n)).astype(np.int64)
    bad = np.abs(out) > NOISE_BOUND
    while bad.any():
        out[bad] = np.rint(rng.normal(0.0, NOISE_SIGMA, int(bad.sum()))).astype(np.int64)
        bad = np.abs(out) > NOISE_BOUND
    return out


def _uniform(ctx, rng) -> np.ndarray:
    return np.stack([rng.integers(0, p.value, ctx.ring_degree, dtype=np.int64) for p in ctx.primes])


def keygen(params: BfvParams, rng: np.random.Generator):
    """(sk, pk, rlk) with the reference's draw order (bfv.py:164-188)."""
    ctx = params.ctx
    m = ctx._modcol
    s_bits = rng.integers(0, 2, ctx.ring_degree, dtype=np.int64)
    s_ntt = ctx.ntt.forward(s_bits[None, :] % m)
    s2 = s_ntt * s_ntt % m
    a = _uniform(ctx, rng)
    e = ctx.ntt.forward(_gauss(rng, ctx.ring_degree)[None, :] % m)
    b = (e - a * s_ntt % m) % m
    comps = []
    wp = 1
    for _ in range(params.l + 1):
        ai = _uniform(ctx, rng)
        ei = ctx.ntt.forward(_gauss(rng, ctx.ring_degree)[None, :] % m)
        k0 = (s2 * ctx.reduce_scalar(wp) % m - (ai * s_ntt % m + ei) % m) % m
        comps.append((RingElem(ctx, k0, Domain.NTT), RingElem(ctx, ai, Domain.NTT)))
        wp *= params.w
    sk = SecretKey(s_bits=s_bits, s_ntt=RingElem(ctx, s_ntt, Domain.NTT),
                   s2_ntt=RingElem(ctx, s2, Domain.NTT))
    pk = PublicKey(RingElem(ctx, b, Domain.NTT), RingElem(ctx, a, Domain.NTT), params.fingerprint)
    return sk, pk, RelinKey(comps, params.w, params.fingerprint)


def encrypt(pk: PublicKey, pt: Plaintext, params: BfvParams, rng: np.random.Generator) -> Ciphertext:
    """u, e1, e2 drawn in the reference's order (bfv.py:201-216)."""
    if pk.fingerprint != params.fingerprint:
        raise ParameterMismatchError("object does not match parameter set")
    if pt.t != params.t:
        raise ParameterMismatchError("plaintext modulus mismatch")
    if pt.poly.shape != (params.ring_degree,) or (pt.poly < 0).any() or (pt.poly >= params.t).any():
        raise EncodingError("plaintext coefficient outside [0, t)")
    ctx = params.ctx
    m = ctx._modcol
    u = rng.integers(0, 2, ctx.ring_degree, dtype=np.int64)
    un = ctx.ntt.forward(u[None, :] % m)
    c = ctx.ntt.inverse(np.concatenate([pk.b_ntt.residues * un % m, pk.a_ntt.residues * un % m]),
                        sel=np.concatenate([np.arange(len(ctx.primes))] * 2))
    k = len(ctx.primes)
    c0, c1 = c[:k], c[k:]
    e1 = _gauss(rng, ctx.ring_degree)
    e2 = _gauss(rng, ctx.ring_degree)
    c0 = (c0 + e1[None, :]) % m
    c1 = (c1 + e2[None, :]) % m
    c0 = (c0 + params.delta_col * (pt.poly[None, :] % m) % m) % m
    return Ciphertext((RingElem(ctx, c0, Domain.COEFF), RingElem(ctx, c1, Domain.COEFF)),
                      params.fingerprint, is_fresh=True)


def encrypt_many(pk: PublicKey, polys: np.ndarray, params: BfvParams, rng: np.random.Generator,
                 chunk: int = 64) -> np.ndarray:
    """Encrypt P plaintext polys -> int64 residues [P][2][K][N].

    Draws (u, e1, e2) per ciphertext in exactly the order of P successive
    `encrypt` calls (bfv.py:201-216); the transforms run batched.
    """
    if pk.fingerprint != params.fingerprint:
        raise ParameterMismatchError("object does not match parameter set")
    polys = np.asarray(polys, dtype=np.int64)
    if (polys < 0).any() or (polys >= params.t).any():
        raise EncodingError("plaintext coefficient outside [0, t)")
    ctx = params.ctx
    n, k = ctx.ring_degree, len(ctx.primes)
    m = ctx._modcol
    P = polys.shape[0]
    us = np.empty((P, n), dtype=np.int64)
    e1s = np.empty((P, n), dtype=np.int64)
    e2s = np.empty((P, n), dtype=np.int64)
    for i in range(P):
        us[i] = rng.integers(0, 2, n, dtype=np.int64)
        e1s[i] = _gauss(rng, n)
        e2s[i] = _gauss(rng, n)
    out = np.empty((P, 2, k, n), dtype=np.int64)
    sel = np.arange(k)
    for s0 in range(0, P, chunk):
        c = min(chunk, P - s0)
        u = (us[s0:s0 + c, None, :] % m[None]).reshape(c * k, n)
        un = ctx.ntt.forward(u, sel=np.tile(sel, c)).reshape(c, k, n)
        prod = np.concatenate([pk.b_ntt.residues[None] * un % m, pk.a_ntt.residues[None] * un % m], axis=1)
        ci = ctx.ntt.inverse(prod.reshape(c * 2 * k, n), sel=np.tile(sel, 2 * c)).reshape(c, 2, k, n)
        c0 = (ci[:, 0] + e1s[s0:s0 + c, None, :]) % m
        c1 = (ci[:, 1] + e2s[s0:s0 + c, None, :]) % m
        c0 = (c0 + params.delta_col[None] * (polys[s0:s0 + c, None, :] % m) % m) % m
        out[s0:s0 + c, 0] = c0
        out[s0:s0 + c, 1] = c1
    return out


def _crt_lift(ctx, res: np.ndarray) -> list:
    q = ctx.q_big
    acc = [0] * ctx.ring_degree
    for i, p in enumerate(ctx.primes):
        big = q // p.value
        w = big * pow(big % p.value, -1, p.value) % q
        acc = [a + int(r) * w for a, r in zip(acc, res[i].tolist())]
    return [a % q for a in acc]


def decrypt(sk: SecretKey, c, params) -> Plaintext:
    """Exact-rounding decryption (bfv.py:239-250)."""
    ctx = params.ctx
    m = ctx._modcol if hasattr(ctx, "_modcol") else ctx.prime_values.reshape(-1, 1)
    ntt = ctx.ntt if hasattr(ctx, "ntt") else RnsContext(ctx.ring_degree, [p.value for p in ctx.primes]).ntt
    ph = c.parts[0].residues + ntt.inverse(ntt.forward(c.parts[1].residues) * sk.s_ntt.residues % m)
    if len(c.parts) == 3:
        ph = ph + ntt.inverse(ntt.forward(c.parts[2].residues) * sk.s2_ntt.residues % m)
    v = _crt_lift(ctx, ph % m)
    q, t = ctx.q_big, params.t
    out = [((2 * x * t + q) // (2 * q)) % t for x in v]
    return Plaintext(np.array(out, dtype=np.int64), t)


# ---------------------------------------------------------------- slots


class SlotVector:
    __slots__ = ("values", "t")

    def __init__(self, values, t: int):
        values = np.asarray(values, dtype=np.int64)
        if (values < 0).any() or (values >= t).any():
            raise EncodingError("slot value outside [0, t)")
        self.values = values
        self.t = t


class SlotEncoder:
    """Slot i = evaluation at zeta^(2i+1) over Z_t (batching.py:41-95)."""

    def __init__(self, t: int, ring_degree: int):
        if not is_prime(t):
            raise UnsupportedParametersError(f"t={t} is not prime")
        if (t - 1) % (2 * ring_degree):
            raise UnsupportedParametersError(f"2N={2 * ring_degree} does not divide t-1={t - 1}")
        self.t = t
        self.n = ring_degree
        self.zeta = primitive_root_2n(t, ring_degree)
        # int64 products below 2^31, chunked int64 below 2^47, else Python ints
        self._tr = _Transform(ring_degree, [t], [self.zeta], obj=t >= (1 << 31))

    def encode(self, v) -> Plaintext:
        values = v.values if isinstance(v, SlotVector) else np.asarray(v)
        if values.shape != (self.n,):
            raise EncodingError("slot vector length != N")
        a = values.reshape(1, self.n)
        if self._tr.obj:
            a = np.array([[int(x) % self.t for x in values]], dtype=object)
        out = self._tr.inverse(a)
        return Plaintext(np.array([int(x) for x in out[0]], dtype=np.int64), self.t)

    def encode_many(self, rows: np.ndarray) -> np.ndarray:
        """Encode a (P, N) batch of slot vectors at once -> (P, N) int64."""
        rows = np.asarray(rows)
        if self._tr.obj:
            a = rows.astype(object) % self.t
        else:
            a = rows.astype(np.int64) % self.t
        tr = self._tr
        sel = np.zeros(len(rows), dtype=np.int64)
        return tr.inverse(a, sel=sel).astype(np.int64)

    def decode(self, pt: Plaintext) -> SlotVector:
        a = np.asarray(pt.poly).reshape(1, self.n)
        if self._tr.obj:
            a = a.astype(object)
        out = self._tr.forward(a)
        return SlotVector(np.array([int(x) for x in out[0]], dtype=np.int64), self.t)
