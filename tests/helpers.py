"""Shared builders for tests: mirror params/keys from golden fixtures."""

from __future__ import annotations

import numpy as np

from paper_1811_00778_b200 import bfv as B


def params_of(meta):
    ctx = B.RnsContext(meta["n"], meta["primes"])
    return B.BfvParams(ctx, meta["t"])


def rlk_from_array(params, arr):
    """golden rlk u32 [D][2][K][N] (reference NTT order) -> mirror RelinKey"""
    ctx = params.ctx
    comps = [
        (B.RingElem(ctx, arr[i, 0].astype(np.int64), B.Domain.NTT),
         B.RingElem(ctx, arr[i, 1].astype(np.int64), B.Domain.NTT))
        for i in range(arr.shape[0])
    ]
    return B.RelinKey(comps, params.w, params.fingerprint)


def ct_from_array(params, arr):
    ctx = params.ctx
    parts = tuple(B.RingElem(ctx, arr[p].astype(np.int64), B.Domain.COEFF) for p in range(arr.shape[0]))
    return B.Ciphertext(parts, params.fingerprint)


def ct_array(c):
    return np.stack([p.residues for p in c.parts]).astype(np.int64)


def tensor_from_array(params, arr, shape, delta=1):
    from paper_1811_00778_b200.engine import CipherTensor

    return CipherTensor(shape=tuple(shape), cts=[ct_from_array(params, a) for a in arr], delta=delta,
                        channel_modulus=params.t)


def layer_dicts(spec, weights):
    """NetworkSpec + weights -> the oracle's list-of-dicts network"""
    out = []
    for layer, w in zip(spec.layers, weights):
        k = layer.kind.value
        d = {"kind": k, "name": layer.name}
        if k == "conv":
            d.update(kernel=layer.kernel, stride=layer.stride, padded=layer.padded,
                     groups=layer.groups, weight_scale=layer.weight_scale, weights=w)
        elif k == "fc":
            d.update(weight_scale=layer.weight_scale, weights=w)
        elif k == "pool":
            d.update(extent=layer.extent, stride=layer.stride)
        out.append(d)
    return out
