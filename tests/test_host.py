"""Host-side logic that needs no GPU: the C-ABI library loads and binds every
declared symbol, counters follow the reference's OpCounter semantics,
network tables and error mapping match the reference."""

import os
import re

import numpy as np
import pytest

import hcnn_oracle as O
from conftest import ROOT

from paper_1811_00778_b200 import _lib, errors, nn
from paper_1811_00778_b200 import engine as E


def header_symbols():
    with open(os.path.join(ROOT, "include", "hcnn_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"\b(hcnn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.hcnn_version().startswith(b"hcnn_b200")


def test_library_is_sm100a_native():
    """The shared object carries sm_100a SASS only (no PTX JIT, no other arch)."""
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_status_codes_map_onto_reference_exceptions():
    assert errors.STATUS[1] is errors.ParameterMismatchError
    assert errors.STATUS[2] is errors.MissingKeyError
    assert errors.STATUS[3] is errors.CapacityError
    assert issubclass(errors.BackendError, errors.HefirError)


def test_network_shapes():
    assert nn.mnist_hcnn().layer_shapes() == [(12, 12, 5), (12, 12, 5), (4, 4, 50), (4, 4, 50), (1, 1, 10)]
    assert nn.cifar10_hcnn().layer_shapes()[-1] == (1, 1, 10)
    assert nn.cifar10_hcnn().layer_shapes()[2] == (16, 16, 32)


def _oracle_counts(h, w, c, layer, weights):
    """scheduled / executed / hadd by the reference's loops (engine.py:206-303)."""
    f, kh, kw, cg = weights.shape
    sh, sw = layer.stride
    ph = (kh - 1) // 2 if layer.padded else 0
    pw = (kw - 1) // 2 if layer.padded else 0
    oh = (h + 2 * ph - kh) // sh + 1
    ow = (w + 2 * pw - kw) // sw + 1
    per = f // layer.groups
    sched = ex = hadd = 0
    for oy in range(oh):
        for ox in range(ow):
            for fi in range(f):
                used = 0
                for ky in range(kh):
                    if not 0 <= oy * sh + ky - ph < h:
                        continue
                    for kx in range(kw):
                        if not 0 <= ox * sw + kx - pw < w:
                            continue
                        for ci in range(cg):
                            sched += 1
                            if weights[fi, ky, kx, ci] != 0:
                                used += 1
                ex += used
                hadd += max(used - 1, 0)
    _ = per
    return sched, ex, hadd


@pytest.mark.parametrize("seed", range(6))
def test_conv_counters_match_reference_loops(seed):
    rng = np.random.default_rng(seed)
    h, w = int(rng.integers(3, 9)), int(rng.integers(3, 9))
    groups = int(rng.choice([1, 2]))
    c = groups * int(rng.integers(1, 3))
    f = groups * int(rng.integers(1, 3))
    k = int(rng.choice([1, 3, 5]))
    if k > min(h, w):
        k = 1
    layer = nn.conv_layer("c", f, (k, k), (int(rng.integers(1, 3)),) * 2, bool(rng.integers(0, 2)), 15,
                          groups=groups)
    weights = rng.integers(-2, 3, (f, k, k, c // groups))
    assert E._conv_counts(h, w, layer, weights) == _oracle_counts(h, w, c, layer, weights)


def test_published_scheduled_counts():
    """MNIST conv1 schedules 18,000 multiplies (test_engine.py:245-256); the
    CIFAR engine-scheduled total is 9,673,600."""
    spec = nn.mnist_hcnn()
    s, _, _ = E._conv_counts(28, 28, spec.layers[0], np.ones((5, 5, 5, 1)))
    assert s == 18000
    s2, _, _ = E._conv_counts(12, 12, spec.layers[2], np.ones((50, 5, 5, 1)))
    assert s2 == 20000
    cifar = nn.cifar10_hcnn()
    shapes = [cifar.input_shape] + cifar.layer_shapes()
    total = 0
    for i, layer in enumerate(cifar.layers):
        hh, ww, cc = shapes[i]
        if nn.kind_of(layer) == "conv":
            total += E._conv_counts(hh, ww, layer, np.ones((layer.filters, 3, 3, cc)))[0]
        elif nn.kind_of(layer) == "fc":
            total += layer.filters * hh * ww * cc
    assert total == 9_673_600


def test_fc_counters():
    w = np.array([[0, 1, 2], [0, 0, 0], [3, 0, 0]])
    assert E._fc_counts(w) == (9, 3, 1)


def test_gpu_context_refuses_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_1811_00778_b200 import bfv as B

    params = B.BfvParams(B.RnsContext(64, [1073643521, 1073479681]), 257)
    with pytest.raises(errors.HefirError):
        E.GpuContext(params)


def test_reduce_model_and_crt_reconstruct():
    model = nn.QuantizedModel(nn.toy_hcnn(), 4, [np.array([[[[300]]]]), None, np.array([[-5, 7]])])
    r = E.reduce_model(model, 257)
    assert r.weights[0].item() == 300 - 257 and r.weights[2].tolist() == [[-5, 7]]
    res = E.ChannelResult(moduli=(257, 65537), batch_size=1)
    v = -123456
    res.add(257, np.array([[v % 257]]))
    res.add(65537, np.array([[v % 65537]]))
    assert E.reconstruct_logits(res, (257, 65537))[0, 0] == v
    with pytest.raises(errors.IncompleteResultError):
        E.reconstruct_logits(E.ChannelResult(moduli=(257, 65537), batch_size=1), (257, 65537))
    assert E.classify_logits([[1, 5, 5], [9, 0, 1]]) == [1, 0]


def test_oracle_is_not_imported_by_the_product():
    import subprocess
    import sys

    code = ("import sys, paper_1811_00778_b200.engine, paper_1811_00778_b200.ops, "
            "paper_1811_00778_b200.bfv; assert 'hcnn_oracle' not in sys.modules")
    subprocess.run([sys.executable, "-c", code], check=True, cwd=ROOT)
    pkg = os.path.join(ROOT, "paper_1811_00778_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            with open(os.path.join(pkg, fn)) as fh:
                assert "hcnn_oracle" not in fh.read(), fn
    _ = O


# ------------------------------------------------------------------ HFIR (host side)


def _hfir():
    from conftest import load_golden

    return load_golden("hfir")


def test_hfir_header_and_errors_match_reference_offsets():
    """Header parsing and the host-side errors of the device HFIR reader follow
    serial.py:53-84 (same classes, same byte offsets) -- no GPU needed."""
    from paper_1811_00778_b200 import bfv as B
    from paper_1811_00778_b200 import hfir
    from paper_1811_00778_b200.errors import FormatError, ParameterMismatchError

    meta, a = _hfir()
    params = B.BfvParams(B.RnsContext(meta["n"], meta["primes"]), meta["t"])
    blob = a["tensor"].tobytes()
    import io

    kind, n, primes, t = hfir.read_header(io.BytesIO(blob))
    assert (kind, n, primes, t) == (hfir.KIND_CIPHER_TENSOR, meta["n"], meta["primes"], meta["t"])
    assert hfir.header_bytes(hfir.KIND_CIPHER_TENSOR, params) == blob[: 4 + 3 + 6 + 8 * len(primes) + 8]
    cases = [
        (b"XFIR" + blob[4:], 0),
        (blob[:4] + b"\x02\x00" + blob[6:], 4),
        (blob[:6] + bytes([hfir.KIND_CIPHERTEXT]) + blob[7:], 6),
        (blob[:10], 10),
    ]
    for bad, off in cases:
        with pytest.raises(FormatError) as ei:
            hfir.load_cipher_tensor_device(bad, params)
        assert ei.value.offset == off
    other = B.BfvParams(B.RnsContext(meta["n"], meta["primes"]), 65537)
    with pytest.raises(ParameterMismatchError):
        hfir.load_cipher_tensor_device(blob, other)


def test_hfir_relin_key_reader_matches_reference_keys():
    """load_relin_key_device keeps the serialised coefficient-domain key; its
    NTT (oracle, reference order) equals the reference's in-memory key."""
    import hcnn_oracle as O

    from paper_1811_00778_b200 import bfv as B
    from paper_1811_00778_b200 import hfir

    meta, a = _hfir()
    params = B.BfvParams(B.RnsContext(meta["n"], meta["primes"]), meta["t"])
    key = hfir.load_relin_key_device(a["rlk_file"].tobytes(), params)
    assert key.coeff.shape == a["rlk"].shape and key.base == params.w
    ctx = O.Context(meta["n"], meta["primes"])
    for i in range(key.coeff.shape[0]):
        for part in range(2):
            got = O.ntt_forward(ctx, key.coeff[i, part].astype(np.int64))
            assert np.array_equal(got, a["rlk"][i, part].astype(np.int64))


def test_plain_c_program_links_and_fails_loudly_without_a_gpu(tmp_path):
    """The C example resolves the in-tree library; without a CUDA device the
    first ABI call returns HCNN_ERR_CUDA (5) instead of computing anything."""
    import struct
    import subprocess

    import torch

    exe = os.path.join(ROOT, "examples", "capi_hsquare")
    if not os.path.exists(exe):
        pytest.skip("example not built")
    ldd = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libhcnn_b200.so =>" in ldd and "not found" not in ldd
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    src = tmp_path / "in.bin"
    with open(src, "wb") as fh:
        fh.write(struct.pack("<IIIQI", 64, 1, 0, 257, 16))
        fh.write(struct.pack("<Q", 1073643521))
    r = subprocess.run([exe, str(src), str(tmp_path / "out.bin")], capture_output=True, text=True)
    assert r.returncode == 5, (r.returncode, r.stderr)


def test_host_narrow_is_exact_and_rejects_out_of_range():
    """hcnn_host_narrow (host-only, no device): int64 residue arrays -> one
    u32 buffer, every thread count; values outside [0, 2^32) are refused."""
    import ctypes

    from paper_1811_00778_b200 import _lib
    from paper_1811_00778_b200.errors import ParameterMismatchError

    rng = np.random.default_rng(3)
    arrs = [rng.integers(0, 1 << 30, (3, 257)).astype(np.int64) for _ in range(11)]
    ptrs = np.array([a.ctypes.data for a in arrs], dtype=np.uintp)
    for threads in (1, 3, 0, 64):
        dst = np.zeros((11, 3, 257), dtype=np.uint32)
        _lib.check(_lib.lib().hcnn_host_narrow(ptrs.ctypes.data, 11, 3 * 257, dst.ctypes.data, threads))
        assert np.array_equal(dst.astype(np.int64), np.stack(arrs))
    arrs[7][2, 5] = -1
    dst = np.zeros((11, 3, 257), dtype=np.uint32)
    with pytest.raises(ParameterMismatchError):
        _lib.check(_lib.lib().hcnn_host_narrow(ptrs.ctypes.data, 11, 3 * 257, dst.ctypes.data, 4))
    # 32-byte aligned rows of a multiple of 8 words: the vector (streaming
    # store) path, including a high word set inside its body
    big = [rng.integers(0, 1 << 32, (4, 1024)).astype(np.int64) for _ in range(5)]
    bp = np.array([a.ctypes.data for a in big], dtype=np.uintp)
    raw = np.zeros(5 * 4096 + 8, dtype=np.uint32)
    off = ((32 - raw.ctypes.data % 32) % 32) // 4
    out = raw[off:off + 5 * 4096]
    _lib.check(_lib.lib().hcnn_host_narrow(bp.ctypes.data, 5, 4096, out.ctypes.data, 2))
    assert np.array_equal(out.reshape(5, 4, 1024).astype(np.int64), np.stack(big))
    big[3][1, 17] = 1 << 32
    with pytest.raises(ParameterMismatchError):
        _lib.check(_lib.lib().hcnn_host_narrow(bp.ctypes.data, 5, 4096, out.ctypes.data, 2))
    _ = ctypes


def test_host_widen_is_exact():
    """hcnn_host_widen (host-only): one u32 buffer -> count int64 arrays (the
    drop-in's result objects), every thread count."""
    from paper_1811_00778_b200 import _lib

    rng = np.random.default_rng(4)
    src = rng.integers(0, 1 << 32, (7, 2 * 257), dtype=np.uint64).astype(np.uint32)
    for threads in (1, 3, 0, 64):
        dst = [np.full((2, 257), -1, dtype=np.int64) for _ in range(7)]
        ptrs = np.array([a.ctypes.data for a in dst], dtype=np.uintp)
        _lib.check(_lib.lib().hcnn_host_widen(src.ctypes.data, 7, 2 * 257, ptrs.ctypes.data, threads))
        assert np.array_equal(np.stack(dst).reshape(7, -1), src.astype(np.int64))



def test_rbasis_crt_identity_in_python_ints():
    """The arithmetic of the relinearisation over R (csrc/relin_rb.cuh,
    k_rb_inv), restated with Python ints at N = 64 with the worst-case
    digits (w - 1) and keys: the negacyclic sums Z = sum_i d_i k~_i (keys
    centred mod q_j) are recovered from their residues mod r0, r1, r2 by
    x~_a = Z (R/r_a)^-1 mod r_a, v = rint(sum_a x~_a / r_a) in float32, and
    Z = sum_a x~_a (R/r_a) - v R, so Z mod q_j equals the reference's
    sum_i d_i k_{i,j} mod q_j (bfv.py:368-404)."""
    r = [894959617, 893255681, 889454593]  # the library's R primes (= 1 mod 2^17, below 2^32/sqrt(23))
    R = r[0] * r[1] * r[2]
    n, D, w = 64, 21, 1 << 16
    q = 1073643521
    rng = np.random.default_rng(11)

    def negacyclic(a, b):
        out = [0] * n
        for i in range(n):
            for j in range(n):
                k = i + j
                if k < n:
                    out[k] += a[i] * b[j]
                else:
                    out[k - n] -= a[i] * b[j]
        return out

    for trial in range(3):
        if trial == 0:  # extreme: every digit w - 1, keys at +-(q - 1) / 2
            digits = [[w - 1] * n for _ in range(D)]
            keys = [[(q - 1) // 2 if (i + j) % 2 else -((q - 1) // 2) for j in range(n)] for i in range(D)]
        else:
            digits = [[int(v) for v in rng.integers(0, w, n)] for _ in range(D)]
            keys = [[int(v) - (q - 1) // 2 for v in rng.integers(0, q, n)] for _ in range(D)]
        Z = [0] * n
        for i in range(D):
            for k, v in enumerate(negacyclic(digits[i], keys[i])):
                Z[k] += v
        assert max(abs(z) for z in Z) * 4 < R  # the host check |Z| <= R / 4
        rinv = [np.float32(1.0 / ra) for ra in r]
        for k in range(n):
            xt = [Z[k] * pow(R // ra, -1, ra) % ra for ra in r]
            f = np.float32(0)
            for a in range(3):
                f = np.float32(f + np.float32(xt[a]) * rinv[a])
            v = int(np.rint(f))
            back = sum(xt[a] * (R // r[a]) for a in range(3)) - v * R
            assert back == Z[k]
            assert back % q == sum(digits[i][kk] * keys[i][(k - kk) % n] * (1 if kk <= k else -1)
                                   for i in range(D) for kk in range(n)) % q


def _tc_bytes(x):
    """little-endian bytes of u32 words (the A rows of tc_bconv.cuh)"""
    return [(int(x) >> (8 * b)) & 0xFF for b in range(4)]


def test_tensor_core_base_conversion_identity_in_python_ints():
    """The byte-split identity behind k_extend_tc / k_scale_tc
    (csrc/tc_bconv.cuh), restated with the kernel's integer
    widths: A[4i+b] = byte b of x~_i, B[4o+e][4i+b] = byte e of
    (2^8b c_io 2^32 mod m_o); four s32 column sums per output (each
    < 2^22), S = sum_e acc_e 2^8e < 2^46.1, one REDC -> the exact residue
    (sum_i x~_i c_io + v c_vo) mod m_o, for worst-case (all-ones) and random
    operands at K = 15 (the largest the 64-byte row takes)."""
    import random

    rnd = random.Random(5)
    primes = [1073479681, 1072496641, 1071513601, 1070727169, 1069219841, 1068564481, 1068433409,
              1068236801, 1065811969, 1065484289, 1064697857, 1063452673, 1063321601, 1063059457,
              1062862849]
    K = 15
    for trial in range(40):
        m = primes[trial % len(primes)]
        minv = (-pow(m, -1, 1 << 32)) % (1 << 32)
        c = [rnd.randrange(m) for _ in range(K)]
        cv = rnd.randrange(m)
        if trial < 4:
            xt = [(1 << 30) - 1] * K  # every byte 0xFF / 0x3F: the largest column sums
            v = 255
        else:
            xt = [rnd.randrange(primes[i]) for i in range(K)]
            v = rnd.randrange(K + 1)
        bcols = [[0] * 64 for _ in range(4)]
        for i in range(K + 1):
            ci = c[i] if i < K else cv
            for b in range(4 if i < K else 1):
                cp = ((ci << (8 * b)) << 32) % m
                for e in range(4):
                    bcols[e][4 * i + b] = (cp >> (8 * e)) & 0xFF
        arow = sum((_tc_bytes(x) for x in xt), []) + [v, 0, 0, 0]
        arow += [0] * (64 - len(arow))
        acc = [sum(a * bb for a, bb in zip(arow, bcols[e])) for e in range(4)]
        assert all(0 <= s < (1 << 22) for s in acc)
        S = acc[0] + (acc[1] << 8) + (acc[2] << 16) + (acc[3] << 24)
        assert S < (1 << 47)
        u = (S * minv) % (1 << 32)
        r = (S + u * m) >> 32
        r = r if r < m else r - m
        assert r == (sum(x * ci for x, ci in zip(xt, c)) + v * cv) % m


def test_tensor_core_digit_lift_identity_in_python_ints():
    """The digits' canonical lift on the tensor cores: column s sums
    byte(s-b) of q/q_i times byte b of x~_i, plus byte s of 2^(32W) - q times
    V; one carry pass gives sum_i x~_i (q/q_i) - V q exactly (mod 2^(32W),
    where the value lies in [0, 2q)), as mw_lift / mw_sub_mq do."""
    import random

    rnd = random.Random(9)
    qs = [1073643521, 1073479681, 1073184769, 1073053697, 1072857089, 1072496641, 1071513601,
          1070727169, 1069219841, 1068564481, 1068433409]
    K = len(qs)
    q = 1
    for p in qs:
        q *= p
    W = (30 * K + 5 + 31) // 32 + 1
    neg = (1 << (32 * W)) - q
    for _ in range(30):
        x = rnd.randrange(q)
        xt = [x * pow(q // p, -1, p) % p for p in qs]
        lift = sum(t * (q // p) for t, p in zip(xt, qs))
        V = lift // q - rnd.randrange(2)  # the fixed-point estimate: v or v - 1
        V = max(V, 0)
        cols = [0] * (4 * W)
        for i, t in enumerate(xt):
            qb = (q // qs[i]).to_bytes(4 * W, "little")
            tb = _tc_bytes(t)
            for b in range(4):
                for s in range(b, 4 * W):
                    cols[s] += tb[b] * qb[s - b]
        nb = neg.to_bytes(4 * W, "little")
        for s in range(4 * W):
            cols[s] += V * nb[s]
        assert max(cols) < (1 << 22)
        words, carry = [], 0
        for w in range(W):
            t = carry + cols[4 * w] + (cols[4 * w + 1] << 8) + (cols[4 * w + 2] << 16) + (cols[4 * w + 3] << 24)
            words.append(t & 0xFFFFFFFF)
            carry = t >> 32
        S = sum(wd << (32 * i) for i, wd in enumerate(words))
        assert S == lift - V * q and 0 <= S < 2 * q
        if S >= q:
            S -= q
        assert S == x
