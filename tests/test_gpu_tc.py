"""Base conversions on the tensor cores (flag TC_BCONV = 32768,
csrc/tc_bconv.cuh): the multiply's Q -> P extension (k_extend) and its exact
t/q scale-and-round (k_scale, both conversions) as u8 x u8 -> s32 tcgen05
MMAs.  Whatever the flag, every output limb must equal the reference's
hmult_raw / hsquare (bfv.py:331-347, 407-443): checked against the integer
kernels on random and extreme inputs and against the pinned oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import hcnn_oracle as O  # noqa: E402
from helpers import ct_array  # noqa: E402

from paper_1811_00778_b200 import _lib  # noqa: E402
from paper_1811_00778_b200 import bfv as B  # noqa: E402
from paper_1811_00778_b200 import engine as E  # noqa: E402
from paper_1811_00778_b200 import ops  # noqa: E402

TC = 32768
Q_TC = 9


def dev(arr):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(arr).astype(np.uint32)).view(np.int32)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32).astype(np.int64)


def _primes(n, k):
    out, c = [], (1 << 30) // (2 * n)
    while len(out) < k:
        p = c * 2 * n + 1
        if p < (1 << 30) and all(p % d for d in range(3, int(p ** 0.5) + 1, 2)):
            out.append(p)
        c -= 1
    return out


def _two_part(primes, n, rng, count):
    """[count][2][K][N] canonical residues; the first rows hold q - 1, 0,
    (q-1)/2 and (q+1)/2 in every limb (lifts at the edges of [0, q) and at the
    centre, where the CRT overflow estimate is decided exactly)"""
    k = len(primes)
    p = np.array(primes, dtype=np.int64)[:, None]
    x = rng.integers(0, 1 << 62, (count, 2, k, n)) % p
    x[0, 0] = p - 1
    x[0, 1] = 0
    x[1, 0] = (p - 1) // 2
    x[1, 1] = (p + 1) // 2 % p
    return x


@pytest.mark.parametrize("n,k,t", [(8192, 11, 5522259017729), (8192, 6, 65537), (1024, 4, 257),
                                   (16384, 11, 5522259017729), (32768, 12, 65537), (4096, 13, 65537),
                                   (8192, 10, 2424833)])
def test_tc_hmult_raw_equals_integer_kernels(n, k, t):
    """hmult_raw (square and general) with the flag on and off agree bit for
    bit; the flag is reported active."""
    E._CTXS.clear()
    primes = _primes(n, k)
    params = B.BfvParams(B.RnsContext(n, primes), t)
    g = E.context_for(params)
    rng = np.random.default_rng(n + k)
    a = dev(_two_part(primes, n, rng, 13))  # >= 12: the tensor-core path's minimum batch
    b = dev(_two_part(primes, n, rng, 13)[::-1])
    base = g.variant() & ~TC
    g.set_variant(base)
    assert _lib.lib().hcnn_ctx_query(g.handle, Q_TC) == 0
    want_sq = host(ops.hmult_raw_device(g, a, a))
    want = host(ops.hmult_raw_device(g, a, b))
    g.set_variant(base | TC)
    assert _lib.lib().hcnn_ctx_query(g.handle, Q_TC) == 1
    g.profile(True)
    got_sq = host(ops.hmult_raw_device(g, a, a))
    names = set(g.profile_read())
    g.profile(False)
    assert {"k_extend_tc", "k_scale_tc"} <= names and "k_scale" not in names, names
    got = host(ops.hmult_raw_device(g, a, b))
    assert np.array_equal(got_sq, want_sq)
    assert np.array_equal(got, want)
    E._CTXS.clear()


@pytest.mark.parametrize("n,k", [(8192, 11), (16384, 8)])
def test_tc_hsquare_vs_oracle(n, k):
    """HSquare (digits of the scaled c2 feed the relinearisation) with the flag
    on equals the oracle's hmult_raw + relinearize on fresh encryptions."""
    E._CTXS.clear()
    primes = _primes(n, k)
    t = 65537
    params = B.BfvParams(B.RnsContext(n, primes), t)
    _, pk, rlk = B.keygen(params, np.random.default_rng(n))
    rng = np.random.default_rng(n + 1)
    cts = [B.encrypt(pk, B.Plaintext(rng.integers(0, t, n), t), params, rng) for _ in range(12)]
    g = E.context_for(params)
    g.set_variant(g.variant() | TC)
    assert _lib.lib().hcnn_ctx_query(g.handle, Q_TC) == 1
    x = dev(np.stack([ct_array(c) for c in cts]))
    g.profile(True)
    got = host(ops.square_device(g, x, rlk))
    names = set(g.profile_read())
    g.profile(False)
    assert "k_scale_tc" in names, names
    op = O.Params(O.Context(n, primes), t)
    orlk = [(k0.residues, k1.residues) for k0, k1 in rlk.components]
    for i in (0, 5, 11):
        c = cts[i]
        ref3 = O.hmult_raw(op, (c.parts[0].residues, c.parts[1].residues))
        assert np.array_equal(got[i], np.stack(O.relinearize(op, ref3, orlk)))
    E._CTXS.clear()


def test_tc_small_batches_take_the_integer_kernels():
    """Below 12 ciphertexts per chunk the integer conversions run (shorter
    latency); results are identical either way."""
    E._CTXS.clear()
    n, k = 8192, 11
    primes = _primes(n, k)
    g = E.context_for(B.BfvParams(B.RnsContext(n, primes), 5522259017729))
    a = dev(_two_part(primes, n, np.random.default_rng(2), 12))
    outs = {}
    for count in (4, 12):
        g.profile(True)
        outs[count] = host(ops.hmult_raw_device(g, a[:count], a[:count]))
        names = set(g.profile_read())
        g.profile(False)
        assert ("k_scale_tc" in names) == (count >= 12) and ("k_scale" in names) == (count < 12), names
    assert np.array_equal(outs[4], outs[12][:4])
    E._CTXS.clear()


def test_tc_unavailable_for_16_primes():
    """K = 16 (4 K + 1 bytes exceed the 64-byte MMA row): the flag is accepted
    and the integer kernels run."""
    E._CTXS.clear()
    n = 1024
    primes = _primes(n, 16)
    params = B.BfvParams(B.RnsContext(n, primes), 65537)
    g = E.context_for(params)
    g.set_variant(g.variant() | TC)
    assert _lib.lib().hcnn_ctx_query(g.handle, Q_TC) == 0
    a = dev(_two_part(primes, n, np.random.default_rng(1), 12))
    g.profile(True)
    ops.hmult_raw_device(g, a, a)
    names = set(g.profile_read())
    g.profile(False)
    assert "k_scale" in names and "k_scale_tc" not in names
    E._CTXS.clear()


RB = 16384
RB_MAC_TC = 65536


def _three_part(primes, n, rng, count):
    k = len(primes)
    p = np.array(primes, dtype=np.int64)[:, None]
    x = rng.integers(0, 1 << 62, (count, 3, k, n)) % p
    x[0, 2] = p - 1  # every digit w - 1: the largest key-switching sums
    x[1, 2] = (p - 1) // 2
    return x


@pytest.mark.parametrize("n,k,count", [(8192, 11, 20), (8192, 12, 131), (16384, 11, 13), (4096, 8, 140)])
def test_tc_relinearisation_mac_equals_integer_mac(n, k, count):
    """The relinearisation multiply-accumulate over R on the tensor cores
    (flag 65536, k_rb_mac_tc) equals the integer k_rb_mac bit for bit, for
    batches that are not multiples of the 128-ciphertext tile."""
    E._CTXS.clear()
    primes = _primes(n, k)
    params = B.BfvParams(B.RnsContext(n, primes), 5522259017729 if n <= 8192 else 65537)
    _, _, rlk = B.keygen(params, np.random.default_rng(k + n))
    x3 = dev(_three_part(primes, n, np.random.default_rng(n + k + count), count))
    g = E.context_for(params)
    _lib.check(_lib.lib().hcnn_ctx_set_option(g.handle, 3, 1), "rb min batch")
    base = (g.variant() | RB) & ~RB_MAC_TC
    g.set_variant(base)
    assert _lib.lib().hcnn_ctx_query(g.handle, 8) == 1
    want = host(ops.relinearize_device(g, x3, rlk))
    g.set_variant(base | RB_MAC_TC)
    g.profile(True)
    got = host(ops.relinearize_device(g, x3, rlk))
    names = set(g.profile_read())
    g.profile(False)
    assert "k_rb_mac_tc" in names and "k_rb_mac" not in names, names
    assert np.array_equal(got, want)
    E._CTXS.clear()


def test_tc_mac_hsquare_vs_oracle():
    """HSquare with every tensor-core path on equals the oracle."""
    E._CTXS.clear()
    n, k, t = 8192, 11, 65537
    primes = _primes(n, k)
    params = B.BfvParams(B.RnsContext(n, primes), t)
    _, pk, rlk = B.keygen(params, np.random.default_rng(3))
    rng = np.random.default_rng(4)
    cts = [B.encrypt(pk, B.Plaintext(rng.integers(0, t, n), t), params, rng) for _ in range(12)]
    g = E.context_for(params)
    g.set_variant(g.variant() | RB | TC | RB_MAC_TC)
    x = dev(np.stack([ct_array(c) for c in cts]))
    got = host(ops.square_device(g, x, rlk))
    op = O.Params(O.Context(n, primes), t)
    orlk = [(k0.residues, k1.residues) for k0, k1 in rlk.components]
    for i in (0, 11):
        c = cts[i]
        ref3 = O.hmult_raw(op, (c.parts[0].residues, c.parts[1].residues))
        assert np.array_equal(got[i], np.stack(O.relinearize(op, ref3, orlk)))
    E._CTXS.clear()
