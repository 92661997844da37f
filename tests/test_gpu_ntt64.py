"""The u64 negacyclic NTT (hcnn_ntt64, csrc/ntt64.cuh) through the C ABI:
bit-exact against the reference's own tables and transform
(tests/golden/ntt64.*: a 62-bit prime and the MNIST t) and against the
pinned oracle at N = 2^13..2^15 (the 2^15 rows on a 2-CTA cluster), with
round trips and edge values; the slot codec on top of it."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import hcnn_oracle as O  # noqa: E402
from conftest import load_golden  # noqa: E402

from paper_1811_00778_b200 import _lib  # noqa: E402


def _prime_1mod(bits, two_n):
    k = ((1 << bits) - 1) // two_n
    while True:
        p = k * two_n + 1
        if p < (1 << bits) and O.is_prime(p):
            return p
        k -= 1


class Ntt64:
    def __init__(self, p, n):
        self.p, self.n = p, n
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().hcnn_codec_create(p, n, 0, ctypes.byref(h)), "hcnn_codec_create")
        self.h = h

    def run(self, rows, inverse):
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(rows, dtype=np.uint64)).view(np.int64)).cuda()
        s = torch.cuda.current_stream().cuda_stream
        _lib.check(_lib.lib().hcnn_ntt64(self.h, ctypes.c_void_p(x.data_ptr()), x.shape[0], int(inverse),
                                         ctypes.c_void_p(s)), "hcnn_ntt64")
        torch.cuda.synchronize()
        return x.cpu().numpy().view(np.uint64)

    def close(self):
        _lib.lib().hcnn_codec_destroy(self.h)


def test_ntt64_reference_golden():
    """Forward: device position i holds the reference's spectral entry brv(i);
    inverse: from that layout back to the reference's coefficients."""
    meta, arrs = load_golden("ntt64")
    for case in meta["cases"]:
        name, p, n = case["name"], case["p"], case["n"]
        rev = O.bitrev_perm(n)
        x, fwd, inv = arrs[name + "_x"], arrs[name + "_fwd"], arrs[name + "_inv"]
        t = Ntt64(p, n)
        assert np.array_equal(t.run(x, False), fwd[:, rev]), name
        # the reference's ntt_inverse of x (x read as a natural-order spectrum)
        assert np.array_equal(t.run(x[:, rev], True), inv), name
        t.close()


@pytest.mark.parametrize("n", [8192, 16384, 32768])
@pytest.mark.parametrize("bits", [62, 50, 30])
def test_ntt64_vs_oracle_and_round_trip(n, bits):
    p = _prime_1mod(bits, 2 * n)
    rng = np.random.default_rng(n + bits)
    x = rng.integers(0, p, (3, n), dtype=np.uint64)
    x[1] = p - 1  # edge rows: all p - 1, all zero
    x[2, : n // 2] = 0
    t = Ntt64(p, n)
    got = t.run(x, False)
    rev = O.bitrev_perm(n)
    want = O.ntt_forward_wide(p, n, x[:2]).astype(np.uint64)
    assert np.array_equal(got[:2], want[:, rev])
    assert np.array_equal(t.run(got, True), x)
    t.close()


def test_ntt64_many_rows_and_small_n():
    for n in (4, 64, 512, 2048):
        p = _prime_1mod(62, 2 * n)
        x = np.random.default_rng(n).integers(0, p, (37, n), dtype=np.uint64)
        t = Ntt64(p, n)
        got = t.run(x, False)
        assert np.array_equal(got[5], O.ntt_forward_wide(p, n, x[5:6]).astype(np.uint64)[0, O.bitrev_perm(n)])
        assert np.array_equal(t.run(got, True), x)
        t.close()
