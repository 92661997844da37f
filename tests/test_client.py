"""The product's host client (keygen / encrypt / encode) reproduces the
reference's bytes for the same seeds, so the GPU box can regenerate every
golden input without the reference tree."""

import hashlib
import json
import os

import numpy as np
import pytest

import hcnn_oracle as O
from conftest import GOLDEN, HAVE_REF, import_reference
from helpers import params_of

from paper_1811_00778_b200 import bfv as B
from paper_1811_00778_b200 import engine as E
from paper_1811_00778_b200 import nn


def sha_cts(arr):
    return hashlib.sha256(np.ascontiguousarray(np.asarray(arr).astype("<u8")).tobytes()).hexdigest()


def test_keygen_matches_golden(golden_small):
    meta, a = golden_small
    params = params_of(meta)
    sk, pk, rlk = B.keygen(params, np.random.default_rng(meta["keys_seed"]))
    assert np.array_equal(np.stack([np.stack([k0.residues, k1.residues]) for k0, k1 in rlk.components]), a["rlk"])
    assert np.array_equal(np.stack([pk.b_ntt.residues, pk.a_ntt.residues]), a["pk"])
    assert np.array_equal(sk.s_bits, a["s_bits"])


def test_encrypt_many_equals_sequential_encrypt():
    params = B.BfvParams(B.RnsContext(256, [1073643521, 1073479681, 1073184769]), 65537)
    _, pk, _ = B.keygen(params, np.random.default_rng(1))
    polys = np.random.default_rng(2).integers(0, 65537, (7, 256))
    r = np.random.default_rng(3)
    seq = np.stack([np.stack([p.residues for p in B.encrypt(pk, B.Plaintext(x, 65537), params, r).parts])
                    for x in polys])
    assert np.array_equal(B.encrypt_many(pk, polys, params, np.random.default_rng(3), chunk=3), seq)


@pytest.mark.parametrize("t,n", [(257, 64), (5522259017729, 1024), (2424833, 64)])
def test_slot_encoder_matches_oracle(t, n):
    enc = B.SlotEncoder(t, n)
    codec = O.SlotCodec(t, n)
    rng = np.random.default_rng(t % 1000)
    s = rng.integers(0, t, n)
    m = enc.encode(s).poly
    assert np.array_equal(m, codec.encode(s))
    assert np.array_equal(enc.decode(B.Plaintext(m, t)).values, s)
    assert np.array_equal(codec.decode(m), s)
    many = enc.encode_many(np.stack([s, s[::-1]]))
    assert np.array_equal(many[1], codec.encode(s[::-1]))


def test_decrypt_roundtrip_and_hsquare_golden(golden_small):
    meta, a = golden_small
    params = params_of(meta)
    sk, pk, _ = B.keygen(params, np.random.default_rng(meta["keys_seed"]))
    c = B.Ciphertext(tuple(B.RingElem(params.ctx, x.astype(np.int64), B.Domain.COEFF) for x in a["hsq"][0]),
                     params.fingerprint)
    op = O.Params(O.Context(meta["n"], meta["primes"]), meta["t"])
    assert np.array_equal(B.decrypt(sk, c, params).poly, O.decrypt(op, sk.s_bits, (c.parts[0].residues, c.parts[1].residues)))


def test_pack_images_reproduces_mnist_golden_input():
    """784 ciphertexts at N=1024 (set-1 primes): same sha256 as the
    reference's pack_images with the golden seeds."""
    with open(os.path.join(GOLDEN, "mnist1024.json")) as fh:
        meta = json.load(fh)
    params = params_of(meta)
    _, pk, _ = B.keygen(params, np.random.default_rng(meta["keys_seed"]))
    irng = np.random.default_rng(meta["image_seed"])
    images = [irng.integers(0, 5, (28, 28, 1)) for _ in range(meta["image_count"])]
    enc = B.SlotEncoder(params.t, params.ring_degree)
    t = E.pack_images(images, E.PackingLayout(len(images), params.ring_degree), enc, pk, params,
                      np.random.default_rng(meta["pack_seed"]), delta=4)
    arr = np.stack([np.stack([p.residues for p in c.parts]) for c in t.cts])
    assert sha_cts(arr) == meta["digests"]["input"]


def test_random_model_is_quantised_and_dense():
    m = nn.random_model(nn.mnist_hcnn(), np.random.default_rng(0))
    assert [None if w is None else w.shape for w in m.weights] == [(5, 5, 5, 1), None, (50, 5, 5, 1), None, (10, 800)]
    for w in m.weights:
        if w is not None:
            assert np.abs(w).max() <= 15
    c = nn.random_model(nn.cifar10_hcnn(), np.random.default_rng(0))
    assert c.weights[0].shape == (32, 3, 3, 3) and c.weights[9].shape == (256, 2048)
    assert np.abs(c.weights[0]).max() <= 10000


@pytest.mark.skipif(not HAVE_REF, reason="reference tree not mounted")
def test_client_matches_live_reference():
    import_reference()
    from hefir import bfv as rb
    from hefir import ring as rr

    primes = [1073643521, 1073479681, 1073184769]
    rp = rb.BfvParams(rr.RnsContext(128, primes), 65537)
    mp = B.BfvParams(B.RnsContext(128, primes), 65537)
    assert mp.fingerprint == rp.fingerprint and mp.l == rp.l and mp.delta == rp.delta
    rsk, rpk, rrlk = rb.keygen(rp, np.random.default_rng(9))
    msk, mpk, mrlk = B.keygen(mp, np.random.default_rng(9))
    for (a0, a1), (b0, b1) in zip(rrlk.components, mrlk.components):
        assert np.array_equal(a0.residues, b0.residues) and np.array_equal(a1.residues, b1.residues)
    x = np.random.default_rng(1).integers(0, 65537, 128)
    rc = rb.encrypt(rpk, rb.Plaintext(x, 65537), rp, np.random.default_rng(5))
    mc = B.encrypt(mpk, B.Plaintext(x, 65537), mp, np.random.default_rng(5))
    for a, b in zip(rc.parts, mc.parts):
        assert np.array_equal(a.residues, b.residues)
    assert np.array_equal(rb.decrypt(rsk, rc, rp).poly, B.decrypt(msk, mc, mp).poly)
