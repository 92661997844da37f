"""Relinearisation over the shared basis R (flag RELIN_RBASIS = 16384,
csrc/relin_rb.cuh): the digit spectra are taken mod three 30-bit primes
instead of mod every q_j and the key-switching sums are brought back to q_j
by an exact centred CRT.  Whatever the flag, every output limb must equal the
reference's relinearize (bfv.py:368-404): checked against the pinned oracle
and against the per-prime kernel on random and extreme inputs (digits all
w - 1, the largest |Z| the bound allows)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import hcnn_oracle as O  # noqa: E402
from helpers import ct_array  # noqa: E402

from paper_1811_00778_b200 import bfv as B  # noqa: E402
from paper_1811_00778_b200 import engine as E  # noqa: E402
from paper_1811_00778_b200 import ops  # noqa: E402

RB = 16384


def rb_context(params):
    """engine context with every batch size on the R path when the flag is set"""
    from paper_1811_00778_b200 import _lib

    g = E.context_for(params)
    _lib.check(_lib.lib().hcnn_ctx_set_option(g.handle, 3, 1), "rb min batch")
    return g


def dev(arr):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(arr).astype(np.uint32)).view(np.int32)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32).astype(np.int64)


def _primes(n, k):
    """k distinct primes = 1 mod 2n below 2^30 (the preset pool's shape)"""
    out, c = [], (1 << 30) // (2 * n)
    while len(out) < k:
        p = c * 2 * n + 1
        if p < (1 << 30) and all(p % d for d in range(3, int(p ** 0.5) + 1, 2)):
            out.append(p)
        c -= 1
    return out


def _three_part(primes, n, rng, count, extreme):
    """[count][3][K][N] canonical residues; extreme rows put c2 = q - 1 (every
    digit w - 1 where w divides the word size) and c2 = q/2 patterns"""
    k = len(primes)
    p = np.array(primes, dtype=np.int64)[:, None]
    x = rng.integers(0, 1 << 62, (count, 3, k, n)) % p
    if extreme:
        x[0, 2] = p - 1
        x[1, 2] = (p - 1) // 2
        x[2, 2] = 0
    return x


@pytest.mark.parametrize("n,log2w,k", [(8192, 16, 11), (8192, 32, 11), (8192, 8, 11), (4096, 16, 11),
                                       (16384, 16, 11), (16384, 32, 11), (32768, 16, 8),
                                       (8192, 16, 12), (8192, 16, 8), (8192, 32, 16)])
def test_rbasis_relinearize_equals_per_prime_kernel(n, log2w, k):
    """k primes of 30 bits, t = the MNIST set-1 modulus: relinearize with the
    flag on and off agree bit for bit on random and extreme 3-part ciphertexts.
    K = 12 gives D = 23, the largest digit count of the R path (its lazy
    64-bit sums are sized for it); w = 2^8 (D = 42) falls back by design."""
    E._CTXS.clear()
    primes = _primes(n, k)
    params = B.BfvParams(B.RnsContext(n, primes), 5522259017729, relin_base=1 << log2w)
    _, _, rlk = B.keygen(params, np.random.default_rng(7 + log2w))
    rng = np.random.default_rng(n + log2w)
    x3 = dev(_three_part(primes, n, rng, 6, True))
    g = rb_context(params)
    base = g.variant() & ~RB
    g.set_variant(base)
    want = host(ops.relinearize_device(g, x3, rlk))
    g.set_variant(base | RB)
    got = host(ops.relinearize_device(g, x3, rlk))
    assert np.array_equal(got, want)
    from paper_1811_00778_b200 import _lib

    # the R path really ran (D <= 23 digits, K >= 8 primes), the per-prime one otherwise
    assert _lib.lib().hcnn_ctx_query(g.handle, 8) == (1 if g.D <= 23 and len(primes) >= 8 else 0)
    E._CTXS.clear()


@pytest.mark.parametrize("n", [4096, 8192, 16384, 32768])
def test_rbasis_hsquare_vs_oracle(n):
    """HSquare with the flag on equals the oracle's hmult_raw + relinearize
    (the reference algorithm) on fresh encryptions, 8 primes."""
    E._CTXS.clear()
    primes = _primes(n, 8)
    t = 65537
    params = B.BfvParams(B.RnsContext(n, primes), t)
    _, pk, rlk = B.keygen(params, np.random.default_rng(n))
    rng = np.random.default_rng(n + 1)
    cts = [B.encrypt(pk, B.Plaintext(rng.integers(0, t, n), t), params, rng) for _ in range(2)]
    g = rb_context(params)
    g.set_variant(g.variant() | RB)
    from paper_1811_00778_b200 import _lib

    assert _lib.lib().hcnn_ctx_query(g.handle, 8) == 1
    x = dev(np.stack([ct_array(c) for c in cts]))
    got = host(ops.square_device(g, x, rlk))
    op = O.Params(O.Context(n, primes), t)
    orlk = [(k0.residues, k1.residues) for k0, k1 in rlk.components]
    for i, c in enumerate(cts):
        ref3 = O.hmult_raw(op, (c.parts[0].residues, c.parts[1].residues))
        assert np.array_equal(got[i], np.stack(O.relinearize(op, ref3, orlk)))
    E._CTXS.clear()


def test_rbasis_key_in_coefficient_domain():
    """A relinearisation key uploaded in the coefficient domain (HFIR form)
    gives the same result over R as the NTT-domain one."""
    from paper_1811_00778_b200 import hfir

    E._CTXS.clear()
    n = 8192
    primes = _primes(n, 8)
    params = B.BfvParams(B.RnsContext(n, primes), 65537)
    _, _, rlk = B.keygen(params, np.random.default_rng(3))
    op = O.Params(O.Context(n, primes), 65537)
    coeff = np.stack([np.stack([O.ntt_inverse(op.ctx, k0.residues), O.ntt_inverse(op.ctx, k1.residues)])
                      for k0, k1 in rlk.components])
    key = hfir.DeviceRelinKey(coeff.astype(np.uint64), params.w, params.fingerprint)
    x3 = dev(_three_part(primes, n, np.random.default_rng(5), 4, True))
    g = rb_context(params)
    g.set_variant(g.variant() & ~RB)
    want = host(ops.relinearize_device(g, x3, rlk))
    g.set_variant(g.variant() | RB)
    from paper_1811_00778_b200 import _lib

    assert _lib.lib().hcnn_ctx_query(g.handle, 8) == 1
    assert np.array_equal(host(ops.relinearize_device(g, x3, key)), want)
    assert np.array_equal(host(ops.relinearize_device(g, x3, rlk)), want)
    E._CTXS.clear()


@pytest.mark.parametrize("n,base", [(16384, 1024 | 4096), (16384, 0), (8192, 0), (4096, 0)])
def test_rbasis_on_other_geometries(n, base):
    """The R path under the non-default geometries of its ring degrees (2^14
    shuffle-tail instead of mixed passes, plain variants) equals the
    per-prime kernel bit for bit."""
    E._CTXS.clear()
    primes = _primes(n, 10)
    params = B.BfvParams(B.RnsContext(n, primes), 65537)
    _, _, rlk = B.keygen(params, np.random.default_rng(9))
    x3 = dev(_three_part(primes, n, np.random.default_rng(10), 3, True))
    g = rb_context(params)
    g.set_variant(base)
    want = host(ops.relinearize_device(g, x3, rlk))
    g.set_variant(base | RB)
    from paper_1811_00778_b200 import _lib

    assert _lib.lib().hcnn_ctx_query(g.handle, 8) == 1
    assert np.array_equal(host(ops.relinearize_device(g, x3, rlk)), want)
    E._CTXS.clear()


def test_small_batches_take_the_per_prime_kernel():
    """Below HCNN_OPT_RB_MIN_BATCH (default 12) relinearisation runs the
    per-prime kernel (faster for a handful of ciphertexts), from it on the R
    path; results are identical."""
    E._CTXS.clear()
    n = 8192
    primes = _primes(n, 11)
    params = B.BfvParams(B.RnsContext(n, primes), 65537)
    _, _, rlk = B.keygen(params, np.random.default_rng(12))
    g = E.context_for(params)
    x3 = dev(_three_part(primes, n, np.random.default_rng(13), 16, True))
    outs = {}
    for count in (4, 16):
        g.profile(True)
        outs[count] = host(ops.relinearize_device(g, x3[:count], rlk))
        names = set(g.profile_read())
        g.profile(False)
        assert ("k_rb_fwd" in names) == (count >= 12) and ("k_relin" in names) == (count < 12), names
    assert np.array_equal(outs[4], outs[16][:4])
    E._CTXS.clear()
