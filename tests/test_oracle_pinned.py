"""The CPU oracle (oracle/hcnn_oracle.py) pinned against the reference.

Every expected value here was produced by the reference itself
(tests/golden/make_golden.py); the last class re-checks the oracle against the
live reference on fresh seeds when /root/reference is mounted.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import hcnn_oracle as O
from conftest import GOLDEN, HAVE_REF, import_reference, load_golden


def _params(meta):
    return O.Params(O.Context(meta["n"], meta["primes"]), meta["t"])


def _rlk(arr):
    return [(arr[i, 0].astype(np.int64), arr[i, 1].astype(np.int64)) for i in range(arr.shape[0])]


def _ct(a):
    return (a[0].astype(np.int64), a[1].astype(np.int64))


class TestRingKAT:
    """Known answers of the reference's ring tests (test_ring.py:76-87, 189-194)."""

    def test_monomial_wraps_negatively(self):
        ctx = O.Context(4, [17])
        x3 = np.array([[0, 0, 0, 1]])
        x1 = np.array([[0, 1, 0, 0]])
        prod = O.ntt_inverse(ctx, O.ntt_forward(ctx, x3) * O.ntt_forward(ctx, x1) % 17)
        assert prod.tolist() == [[16, 0, 0, 0]]

    def test_difference_of_squares(self):
        ctx = O.Context(4, [17])
        a = np.array([[1, 1, 0, 0]])
        b = np.array([[1, 16, 0, 0]])
        prod = O.ntt_inverse(ctx, O.ntt_forward(ctx, a) * O.ntt_forward(ctx, b) % 17)
        assert prod.tolist() == [[1, 0, 16, 0]]

    def test_crt_known_answers(self):
        assert O.crt_combine([4, 4], [17, 13]) == 4
        assert O.crt_combine([0, 4], [3, 5]) == 9

    @pytest.mark.parametrize("n", [8, 16, 64])
    def test_ntt_product_matches_schoolbook(self, n):
        primes = [1073643521, 1073479681]
        ctx = O.Context(n, primes)
        rng = np.random.default_rng(n)
        a = np.stack([rng.integers(0, p, n) for p in primes])
        b = np.stack([rng.integers(0, p, n) for p in primes])
        got = O.ntt_inverse(ctx, O.ntt_forward(ctx, a) * O.ntt_forward(ctx, b) % ctx.mods)
        for r, p in enumerate(primes):
            exp = [0] * n
            for i in range(n):
                for j in range(n):
                    v = int(a[r, i]) * int(b[r, j])
                    if i + j >= n:
                        exp[i + j - n] -= v
                    else:
                        exp[i + j] += v
            assert got[r].tolist() == [e % p for e in exp]

    def test_kronecker_matches_schoolbook(self):
        rng = np.random.default_rng(5)
        n = 16
        a = [int(x) for x in rng.integers(0, 1 << 40, n)]
        b = [int(x) for x in rng.integers(0, 1 << 40, n)]
        got = O.negacyclic_exact(a, b, n, 2 * 40 + 6)
        exp = [0] * n
        for i in range(n):
            for j in range(n):
                if i + j >= n:
                    exp[i + j - n] -= a[i] * b[j]
                else:
                    exp[i + j] += a[i] * b[j]
        assert got == exp

    def test_round_half_away_identity(self):
        """round(t d / q) == floor((t d + (q-1)/2) / q) for odd q, any sign."""
        rng = np.random.default_rng(7)
        q = 1073643521 * 1073479681
        t = 257
        for _ in range(2000):
            d = int(rng.integers(-(1 << 62), 1 << 62)) * int(rng.integers(1, 1 << 20))
            assert O.round_half_away_div(t * d, q) == (t * d + (q - 1) // 2) // q


class TestSmallGolden:
    def test_ntt_forward(self, golden_small):
        meta, a = golden_small
        ctx = O.Context(meta["n"], meta["primes"])
        assert np.array_equal(O.ntt_forward(ctx, a["ntt_in"].astype(np.int64)), a["ntt_out"])

    def test_keygen_reproduces_reference_keys(self, golden_small):
        meta, a = golden_small
        s, pk, rlk = O.keygen(_params(meta), np.random.default_rng(meta["keys_seed"]))
        assert np.array_equal(np.stack([np.stack(c) for c in rlk]), a["rlk"])
        assert np.array_equal(np.stack(pk), a["pk"])
        assert np.array_equal(s, a["s_bits"])

    def test_hmult_raw_relin_hsquare(self, golden_small):
        meta, a = golden_small
        pr = _params(meta)
        rlk = _rlk(a["rlk"])
        for i in range(a["cts"].shape[0]):
            c = _ct(a["cts"][i])
            raw = O.hmult_raw(pr, c)
            assert np.array_equal(np.stack(raw), a["raw"][i]), i
            assert np.array_equal(np.stack(O.relinearize(pr, raw, rlk)), a["hsq"][i]), i
        gen = O.hmult_raw(pr, _ct(a["cts"][0]), _ct(a["cts"][1]))
        assert np.array_equal(np.stack(gen), a["gen_raw"])
        assert np.array_equal(np.stack(O.relinearize(pr, gen, rlk)), a["gen_hmult"])

    def test_layers_and_counters(self, golden_small):
        meta, a = golden_small
        pr = _params(meta)
        x = O.Tensor((5, 5, 2), [_ct(c) for c in a["tensor_in"]], 4)
        cases = {
            "conv_pad_s1": ((3, 3), (1, 1), True, 1),
            "conv_s2_g2": ((3, 3), (2, 2), False, 2),
            "conv_pad_s2_g2": ((3, 3), (2, 2), True, 2),
        }
        for name, (k, st, pad, groups) in cases.items():
            cnt = O.Counter()
            out = O.conv(pr, x, k, st, pad, groups, 15, a[name + "_w"], cnt)
            assert list(out.shape) == meta["counters"][name]["shape"]
            assert np.array_equal(np.stack([np.stack(c) for c in out.cts]), a[name + "_out"]), name
            for f in ("mult_plain_scheduled", "mult_plain_executed", "mult_plain_skipped", "hadd"):
                assert getattr(cnt, f) == meta["counters"][name][f], (name, f)
        cnt = O.Counter()
        out = O.pool(pr, x, 2, (2, 2), cnt)
        assert np.array_equal(np.stack([np.stack(c) for c in out.cts]), a["pool_out"])
        assert cnt.hadd == meta["counters"]["pool"]["hadd"]
        cnt = O.Counter()
        out = O.fc(pr, x, a["fc_w"], 15, cnt)
        assert np.array_equal(np.stack([np.stack(c) for c in out.cts]), a["fc_out"])
        assert cnt.mult_plain_skipped == meta["counters"]["fc"]["mult_plain_skipped"]

    def test_toy_network(self, golden_small):
        meta, a = golden_small
        pr = _params(meta)
        layers = [
            {"kind": "conv", "name": "conv1", "kernel": (3, 3), "stride": (2, 2), "padded": False,
             "groups": 1, "weight_scale": 15, "weights": a["toy_w_conv1"]},
            {"kind": "square", "name": "square1"},
            {"kind": "fc", "name": "fc", "weight_scale": 15, "weights": a["toy_w_fc"]},
        ]
        seen = {}
        cnt = O.Counter()
        x = O.Tensor((8, 8, 1), [_ct(c) for c in a["toy_in"]], 4)
        out = O.network(pr, x, layers, _rlk(a["rlk"]), cnt,
                        hook=lambda n, t: seen.__setitem__(n, np.stack([np.stack(c) for c in t.cts])))
        for name in ("conv1", "square1", "fc"):
            assert np.array_equal(seen[name], a["toy_" + name]), name
        assert cnt.__dict__ == meta["toy_counter"]
        # decrypted slots == the reference's decrypted values == plaintext net mod t
        codec = O.SlotCodec(pr.t, pr.ctx.n)
        vals = np.stack([codec.decode(O.decrypt(pr, a["s_bits"].astype(np.int64), c))[:5] for c in out.cts]).T
        assert np.array_equal(vals, a["toy_decrypted"])
        plain = np.stack([np.array(O.plain_forward(layers, im)).reshape(-1) for im in a["toy_images"]])
        assert np.array_equal(vals, (plain.astype(object) % pr.t).astype(np.int64))


def test_n1024_hsquare_golden(golden_n1024):
    meta, a = golden_n1024
    pr = _params(meta)
    _, _, rlk = O.keygen(pr, np.random.default_rng(meta["keys_seed"]))
    rl = np.stack([np.stack(c) for c in rlk])
    assert hashlib.sha256(rl.astype("<u8").tobytes()).hexdigest() == meta["digests"]["rlk"]
    assert np.array_equal(np.stack(O.hmult_raw(pr, _ct(a["cts"][0]))), a["raw0"])
    for i in (0, 2):  # one random, one edge-value ciphertext
        assert np.array_equal(np.stack(O.hsquare(pr, _ct(a["cts"][i]), rlk)), a["hsq"][i])


def test_cifar_modulus_layers(golden_cifar64):
    meta, a = golden_cifar64
    pr = _params(meta)
    _, _, rlk = O.keygen(pr, np.random.default_rng(meta["keys_seed"]))
    x = O.Tensor((4, 4, 3), [_ct(c) for c in a["tin"]], 255)
    cnt = O.Counter()
    c1 = O.conv(pr, x, (3, 3), (1, 1), True, 1, 10000, a["w"], cnt)
    assert np.array_equal(np.stack([np.stack(c) for c in c1.cts]), a["conv"])
    s1 = O.Tensor(c1.shape, [O.hsquare(pr, c, rlk) for c in c1.cts[:6]], c1.delta)
    assert np.array_equal(np.stack([np.stack(c) for c in s1.cts]), a["square"][:6])
    sq = O.Tensor(c1.shape, [_ct(c) for c in a["square"]], c1.delta ** 2)
    p1 = O.pool(pr, sq, 2, (2, 2), cnt)
    assert np.array_equal(np.stack([np.stack(c) for c in p1.cts]), a["pool"])


def test_mnist1024_golden_is_self_consistent():
    """The fixture model's plaintext logits equal the reference's decrypted
    logits (certified model, no wrap mod t)."""
    with open(os.path.join(GOLDEN, "mnist1024.json")) as fh:
        meta = json.load(fh)
    t = meta["t"]
    dec = np.array(meta["decrypted"], dtype=object)
    plain = np.array(meta["plain"], dtype=object)
    assert ((plain % t) == dec).all()
    assert meta["counter"]["hsquare"] == 720 + 800
    assert meta["counter"]["mult_plain_scheduled"] == 18000 + 20000 + 8000


@pytest.mark.skipif(not HAVE_REF, reason="reference tree not mounted")
class TestAgainstLiveReference:
    def test_hsquare_fresh_seeds(self):
        hefir = import_reference()
        from hefir import bfv, presets, ring

        primes = list(presets.RNS_PRIME_POOL[:5])
        ctx = ring.RnsContext(128, primes)
        params = bfv.BfvParams(ctx, 65537)
        for seed in (1, 2):
            sk, pk, rlk = bfv.keygen(params, np.random.default_rng(seed))
            rng = np.random.default_rng(seed + 10)
            c = bfv.encrypt(pk, bfv.Plaintext(rng.integers(0, 65537, 128), 65537), params, rng)
            ref = bfv.hsquare(c, rlk, params)
            pr = O.Params(O.Context(128, primes), 65537)
            orlk = [(k0.residues, k1.residues) for k0, k1 in rlk.components]
            got = O.hsquare(pr, (c.parts[0].residues, c.parts[1].residues), orlk)
            assert np.array_equal(np.stack(got), np.stack([p.residues for p in ref.parts]))
            _ = hefir

    def test_relin_base_2_8_and_2_32(self):
        import_reference()
        from hefir import bfv, presets, ring

        primes = list(presets.RNS_PRIME_POOL[:4])
        ctx = ring.RnsContext(64, primes)
        for w in (1 << 8, 1 << 32):
            params = bfv.BfvParams(ctx, 257, relin_base=w)
            sk, pk, rlk = bfv.keygen(params, np.random.default_rng(3))
            rng = np.random.default_rng(4)
            c = bfv.encrypt(pk, bfv.Plaintext(rng.integers(0, 257, 64), 257), params, rng)
            ref = bfv.hsquare(c, rlk, params)
            pr = O.Params(O.Context(64, primes), 257, w)
            orlk = [(k0.residues, k1.residues) for k0, k1 in rlk.components]
            got = O.hsquare(pr, (c.parts[0].residues, c.parts[1].residues), orlk)
            assert np.array_equal(np.stack(got), np.stack([p.residues for p in ref.parts]))


def test_hmult_plain_golden():
    """Oracle hmult_plain (scalar and NTT paths, 2- and 3-part) against the
    reference's outputs (tests/golden/plain.*)."""
    from conftest import load_golden

    meta, a = load_golden("plain")
    for tag in ("s", "m"):
        pr = _params(meta[tag])
        cts = a[f"{tag}_cts"]
        for k, pt in enumerate(a[f"{tag}_pts"]):
            out = np.stack([np.stack(O.hmult_plain(pr, tuple(c.astype(np.int64)), pt)) for c in cts])
            if tag == "s":
                assert np.array_equal(out, a["s_out"][k]), k
            else:
                assert hashlib.sha256(out.astype("<u8").tobytes()).hexdigest() == meta["m"]["out_sha"][k], k
        raw3 = tuple(p.astype(np.int64) for p in a[f"{tag}_raw3"])
        for k, pt in enumerate(a[f"{tag}_pts"][:2]):
            out3 = np.stack(O.hmult_plain(pr, raw3, pt))
            if tag == "s":
                assert np.array_equal(out3, a["s_out3"][k])
            else:
                assert hashlib.sha256(out3.astype("<u8").tobytes()).hexdigest() == meta["m"]["out3_sha"][k]


def test_wide_prime_ntt_golden():
    """The oracle's u64 NTT (62-bit primes and the 43-bit MNIST t) equals the
    reference's own tables and transform (tests/golden/ntt64.*, generated by
    running hefir's NttPlan + transform_rows on Python ints)."""
    meta, arrs = load_golden("ntt64")
    for case in meta["cases"]:
        if case["n"] > 1024:
            continue  # the object-dtype oracle is slow at 2^13; the GPU tests cover those rows
        name, p, n = case["name"], case["p"], case["n"]
        x = arrs[name + "_x"]
        assert np.array_equal(O.ntt_forward_wide(p, n, x).astype(np.uint64), arrs[name + "_fwd"]), name
        assert np.array_equal(O.ntt_inverse_wide(p, n, x).astype(np.uint64), arrs[name + "_inv"]), name
        back = O.ntt_inverse_wide(p, n, O.ntt_forward_wide(p, n, x))
        assert np.array_equal(back.astype(np.uint64), x), name
