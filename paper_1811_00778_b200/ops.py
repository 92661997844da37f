"""Per-ciphertext GPU drop-ins for the reference's bfv multiplication path,
plus batched device-tensor entry points used by tests and the microbench.

    hsquare(c, rlk, params)          bfv.py:435-443
    hmult(c1, c2, rlk, params)       bfv.py:419-432
    hmult_raw(c1, c2, params)        bfv.py:407-416
    relinearize(parts3, rlk, params) bfv.py:368-404
    hmult_plain(c, pt, params)       bfv.py:301-318
    hadd(c1, c2)                     bfv.py:264-274  (via params)
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .engine import GpuContext, context_for, _ptr
from .errors import EncodingError, MissingKeyError, ParameterMismatchError


def _check(params, fp):
    if params.fingerprint != fp:
        raise ParameterMismatchError("object does not match parameter set")


def _stack(cts, g: GpuContext, parts: int) -> torch.Tensor:
    host = np.empty((len(cts), parts, g.K, g.N), dtype=np.uint32)
    for i, c in enumerate(cts):
        for p in range(parts):
            host[i, p] = c.parts[p].residues
    return torch.from_numpy(host.view(np.int32)).to(f"cuda:{g.device}")


def _unstack(data: torch.Tensor, like, params) -> list:
    torch.cuda.current_stream(data.device).synchronize()
    res = data.cpu().numpy().view(np.uint32).astype(np.int64)
    el = like.parts[0]
    out = []
    for i in range(res.shape[0]):
        parts = tuple(type(el)(el.ctx, np.ascontiguousarray(res[i, p]), el.domain)
                      for p in range(res.shape[1]))
        out.append(type(like)(parts=parts, fingerprint=params.fingerprint))
    return out


# ------------------------------------------------------------- device batches


def square_device(g: GpuContext, x: torch.Tensor, rlk) -> torch.Tensor:
    out = g.empty(x.shape[0])
    g.set_relin_key(rlk)
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_square(g.handle, _ptr(x), _ptr(out), x.shape[0]), "hcnn_square")
    return out


def hmult_raw_device(g: GpuContext, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    out = g.empty(a.shape[0], parts=3)
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_hmult_raw(g.handle, _ptr(a), _ptr(b), _ptr(out), a.shape[0]),
               "hcnn_hmult_raw")
    return out


def hmult_device(g: GpuContext, a: torch.Tensor, b: torch.Tensor, rlk) -> torch.Tensor:
    out = g.empty(a.shape[0])
    g.set_relin_key(rlk)
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_hmult(g.handle, _ptr(a), _ptr(b), _ptr(out), a.shape[0]), "hcnn_hmult")
    return out


def relinearize_device(g: GpuContext, x3: torch.Tensor, rlk) -> torch.Tensor:
    out = g.empty(x3.shape[0])
    g.set_relin_key(rlk)
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_relinearize(g.handle, _ptr(x3), _ptr(out), x3.shape[0]),
               "hcnn_relinearize")
    return out


def hadd_device(g: GpuContext, a: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    out = g.empty(a.shape[0])
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_hadd(g.handle, _ptr(a), _ptr(b), _ptr(out), a.shape[0]), "hcnn_hadd")
    return out


def ntt_device(g: GpuContext, rows: torch.Tensor, limbs: int, prime_offset: int = 0,
               inverse: bool = False) -> torch.Tensor:
    """In place on a contiguous int32 [R, N] tensor; row r uses prime
    prime_offset + r % limbs (Q primes first, then the auxiliary P primes)."""
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_ntt(g.handle, _ptr(rows), rows.numel() // g.N, limbs, prime_offset,
                                   int(inverse)), "hcnn_ntt")
    return rows


def mul_plain_device(g: GpuContext, x: torch.Tensor, centered) -> torch.Tensor:
    """x [n][2][K][N] times the plaintext with centred coefficients `centered`."""
    pt = np.ascontiguousarray(np.asarray(centered, dtype=np.int64).reshape(-1))
    if pt.size != g.N:
        raise ParameterMismatchError("plaintext length != ring degree")
    out = g.empty(x.shape[0])
    g.bind_stream()
    _lib.check(_lib.lib().hcnn_mul_plain(g.handle, _ptr(x), pt.ctypes.data, _ptr(out), x.shape[0]),
               "hcnn_mul_plain")
    return out


# ------------------------------------------------------------- per-ciphertext


def hmult_plain(c, pt, params):
    """Multiply by a plaintext lifted at its centred representative
    (bfv.py:301-318): scalar path for constants, NTT path otherwise."""
    _check(params, c.fingerprint)
    if pt.t != params.t:
        raise ParameterMismatchError("plaintext modulus mismatch")
    poly = np.asarray(pt.poly)
    if poly.shape != (params.ring_degree,):
        raise EncodingError("plaintext length != ring degree")
    if (poly < 0).any() or (poly >= params.t).any():
        raise EncodingError("plaintext coefficient outside [0, t)")
    half = params.t // 2
    centered = np.where(poly > half, poly - params.t, poly)
    g = context_for(params)
    nparts = len(c.parts)
    x = _stack([c], g, nparts).reshape(-1, g.K, g.N)
    if nparts % 2:  # the kernel takes part pairs: pad a 3-part ct with a zero part
        x = torch.cat([x, torch.zeros_like(x[:1])])
    out = mul_plain_device(g, x.reshape(-1, 2, g.K, g.N), centered).reshape(-1, g.K, g.N)[:nparts]
    torch.cuda.current_stream(out.device).synchronize()
    res = out.cpu().numpy().view(np.uint32).astype(np.int64)
    el = c.parts[0]
    parts = tuple(type(el)(el.ctx, np.ascontiguousarray(res[p]), el.domain) for p in range(nparts))
    return type(c)(parts=parts, fingerprint=params.fingerprint)


def hsquare(c, rlk, params):
    _check(params, c.fingerprint)
    if rlk is None:
        raise MissingKeyError("relinearization key required for hsquare")
    g = context_for(params)
    like = c  # results come back in the caller's Ciphertext / RingElem classes
    if len(c.parts) == 3:
        c = relinearize(c.parts, rlk, params)
    return _unstack(square_device(g, _stack([c], g, 2), rlk), like, params)[0]


def hmult_raw(c1, c2, params):
    _check(params, c1.fingerprint)
    if c1.fingerprint != c2.fingerprint:
        raise ParameterMismatchError("ciphertexts from different parameter sets")
    if len(c1.parts) != 2 or len(c2.parts) != 2:
        raise ParameterMismatchError("hmult_raw expects 2-part inputs")
    g = context_for(params)
    a = _stack([c1], g, 2)
    b = a if c2 is c1 else _stack([c2], g, 2)
    return _unstack(hmult_raw_device(g, a, b), c1, params)[0]


def hmult(c1, c2, rlk, params):
    _check(params, c1.fingerprint)
    if c1.fingerprint != c2.fingerprint:
        raise ParameterMismatchError("ciphertexts from different parameter sets")
    if rlk is None:
        raise MissingKeyError("relinearization key required for hmult")
    if len(c1.parts) == 3:
        c1 = relinearize(c1.parts, rlk, params)
    if len(c2.parts) == 3:
        c2 = relinearize(c2.parts, rlk, params)
    g = context_for(params)
    a = _stack([c1], g, 2)
    b = a if (c2 is c1 or c1.parts is c2.parts) else _stack([c2], g, 2)
    return _unstack(hmult_device(g, a, b, rlk), c1, params)[0]


class _Parts:
    """A bare holder of ciphertext parts (what _stack reads)."""

    def __init__(self, parts):
        self.parts = tuple(parts)


def _ciphertext_class_for(elem):
    """The Ciphertext class that goes with the caller's RingElem class: the
    reference's bfv.Ciphertext when the parts are hefir RingElems (hefir.ring ->
    hefir.bfv), else this package's mirror."""
    import importlib
    import sys

    mod = type(elem).__module__
    pkg = mod.rsplit(".", 1)[0] if "." in mod else ""
    if pkg and (pkg + ".bfv" in sys.modules or mod == pkg + ".ring"):
        try:
            cls = getattr(importlib.import_module(pkg + ".bfv"), "Ciphertext", None)
            if cls is not None:
                return cls
        except ImportError:
            pass
    from .bfv import Ciphertext

    return Ciphertext


def relinearize(parts3, rlk, params):
    """bfv.relinearize (bfv.py:368-404): 3 parts -> a 2-part ciphertext in the
    caller's classes."""
    if rlk is None:
        raise MissingKeyError("relinearization key required")
    _check(params, rlk.fingerprint)
    g = context_for(params)
    out = relinearize_device(g, _stack([_Parts(parts3)], g, 3), rlk)
    el = parts3[0]
    torch.cuda.current_stream(out.device).synchronize()
    res = out.cpu().numpy().view(np.uint32).astype(np.int64)
    parts = tuple(type(el)(el.ctx, np.ascontiguousarray(res[0, p]), el.domain) for p in range(2))
    return _ciphertext_class_for(el)(parts=parts, fingerprint=params.fingerprint)
