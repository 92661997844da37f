"""Round-2 robustness checks of the CUDA path: the integer convolution kernels
that the FP64 path normally hides (k_conv for |w| >= 2^22, k_conv_sw for
filters whose FP64 weight table exceeds shared memory), launches tiled past
the 65,535-block grid limit, stream switches that share the context
workspace, the decrypt-key cache after GPU keygen, and input validation of
the serving loop.  Expected values: the pinned oracle (oracle/) or plain
numpy modular arithmetic on the same inputs."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import hcnn_oracle as O  # noqa: E402

from paper_1811_00778_b200 import bfv as B  # noqa: E402
from paper_1811_00778_b200 import engine as E  # noqa: E402
from paper_1811_00778_b200 import nn, ops  # noqa: E402
from paper_1811_00778_b200.errors import ParameterMismatchError  # noqa: E402

PRIMES = [1073643521, 1073479681, 1073184769]


def _rand_cts(rng, count, primes, n):
    return np.stack([np.stack([np.stack([rng.integers(0, p, n) for p in primes]) for _ in range(2)])
                     for _ in range(count)])


def _conv_vs_oracle(h, w, c, f, k, weights, n=64, primes=PRIMES, seed=0):
    t = 65537
    params = B.BfvParams(B.RnsContext(n, primes), t)
    op = O.Params(O.Context(n, primes), t)
    rng = np.random.default_rng(seed)
    x = _rand_cts(rng, h * w * c, primes, n)
    layer = nn.conv_layer("c", f, (k, k), (1, 1), False, 15)
    tin = E.from_residues(x.astype(np.uint64), (h, w, c), 1, t, params)
    counter = E.OpCounter()
    got = E.eval_conv(tin, layer, weights, params, counter).residues().astype(np.int64)
    ot = O.Tensor((h, w, c), [(cc[0], cc[1]) for cc in x], 1)
    oc = O.Counter()
    ref = O.conv(op, ot, (k, k), (1, 1), False, 1, 15, weights, oc)
    assert np.array_equal(got, np.stack([np.stack(cc) for cc in ref.cts]))
    assert counter.mult_plain_executed == oc.mult_plain_executed and counter.hadd == oc.hadd


def test_conv_general_residue_kernel_large_weights():
    """|w| up to 2^40 (no FP64 table, no u16 table): k_conv with per-limb
    weight residues (ring.py:199-207 with w reduced mod p_i)."""
    rng = np.random.default_rng(5)
    w = rng.integers(-(1 << 40), 1 << 40, (4, 3, 3, 2))
    w[0, 0, 0, 0] = 0  # skipped tap
    w[1, 1, 1, 1] = (1 << 22)
    _conv_vs_oracle(5, 6, 2, 4, 3, w, seed=1)


def test_conv_small_weight_kernel_when_fp64_table_exceeds_smem():
    """3x3x1024 filters: the FP64 weight table (> 96 KB) does not fit, the
    biased-u16 kernel k_conv_sw runs."""
    rng = np.random.default_rng(6)
    w = rng.integers(-15, 16, (2, 3, 3, 1024))
    _conv_vs_oracle(3, 3, 1024, 2, 3, w, seed=2)


def test_conv_and_pool_tiled_past_65535_blocks():
    """260x260 maps: a 1x1 convolution and a 2x2/stride-1 pool both need more
    than 65,535 output blocks; the launches are tiled."""
    n, primes, t = 64, PRIMES[:2], 65537
    params = B.BfvParams(B.RnsContext(n, primes), t)
    h = w = 260
    rng = np.random.default_rng(7)
    mods = np.array(primes, dtype=np.int64)[:, None]
    x = (rng.integers(0, 1 << 30, (h * w, 2, 2, n)) % mods).astype(np.int64)
    tin = E.from_residues(x.astype(np.uint64), (h, w, 1), 1, t, params)
    layer = nn.conv_layer("c", 1, (1, 1), (1, 1), False, 15)
    got = E.eval_conv(tin, layer, np.array([[[[-7]]]]), params, E.OpCounter()).residues().astype(np.int64)
    assert np.array_equal(got, (x * -7) % mods)
    pool = nn.pool_layer("p", 2, 1)
    got = E.eval_pool(tin, pool, params, E.OpCounter()).residues().astype(np.int64)
    xm = x.reshape(h, w, 2, 2, n)
    exp = (xm[:-1, :-1] + xm[1:, :-1] + xm[:-1, 1:] + xm[1:, 1:]) % mods
    assert got.shape[0] == 259 * 259 > 65535
    assert np.array_equal(got, exp.reshape(-1, 2, 2, n))


def test_stream_switch_orders_the_shared_workspace():
    """Squares issued on two torch streams back to back (no host sync in
    between, the second batch larger so the workspace is regrown) equal the
    same squares issued on one stream."""
    n, primes, t = 1024, [1073643521, 1073479681, 1073184769, 1073053697], 65537
    params = B.BfvParams(B.RnsContext(n, primes), t)
    _, _, rlk = B.keygen(params, np.random.default_rng(8))
    g = E.context_for(params)
    rng = np.random.default_rng(9)
    a = torch.from_numpy(_rand_cts(rng, 24, primes, n).astype(np.uint32).view(np.int32)).cuda()
    b = torch.from_numpy(_rand_cts(rng, 96, primes, n).astype(np.uint32).view(np.int32)).cuda()
    ref_a = ops.square_device(g, a, rlk).clone()
    ref_b = ops.square_device(g, b, rlk).clone()
    torch.cuda.synchronize()
    g.set_workspace_limit(1 << 20)  # force chunking and regrowth paths
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s1):
            oa = ops.square_device(g, a, rlk)
        with torch.cuda.stream(s2):
            ob = ops.square_device(g, b, rlk)
        torch.cuda.synchronize()
        assert torch.equal(oa, ref_a) and torch.equal(ob, ref_b)
    g.set_workspace_limit(6 << 30)


def test_decrypt_after_gpu_keygen_uses_the_callers_key():
    """decrypt with key A, keygen_device installs key B, decrypt with A again:
    the result is still A's decryption (the device key cache follows keygen)."""
    n, primes, t = 64, [1073643521, 1073479681, 1073184769, 1073053697], 257
    params = B.BfvParams(B.RnsContext(n, primes), t)
    skA, pkA, _ = B.keygen(params, np.random.default_rng(10))
    m = np.random.default_rng(11).integers(0, t, n)
    c = B.encrypt(pkA, B.Plaintext(m, t), params, np.random.default_rng(12))
    x = E.from_residues(np.stack([p.residues for p in c.parts])[None].astype(np.uint64), (1, 1, 1), 1, t, params)
    assert np.array_equal(E.decrypt_device(x, skA, params).cpu().numpy()[0], m)
    E.keygen_device(params, np.random.default_rng(13))
    assert np.array_equal(E.decrypt_device(x, skA, params).cpu().numpy()[0], m)


def test_serving_loop_rejects_a_short_batch():
    n, primes, t = 64, [1073643521, 1073479681, 1073184769, 1073053697], 257
    params = B.BfvParams(B.RnsContext(n, primes), t)
    _, _, rlk = B.keygen(params, np.random.default_rng(14))
    model = nn.random_model(nn.toy_hcnn(), np.random.default_rng(15))
    short = torch.zeros((63, 2, 4, n), dtype=torch.int32).pin_memory()  # (8, 8, 1) needs 64
    for bands in (1, 6):
        with pytest.raises(ParameterMismatchError):
            E.eval_network_stream([short], model, rlk, params, (8, 8, 1), 4, bands=bands)


def test_library_pool_leaves_the_default_pool_alone():
    """The library allocates from its own memory pool: creating a context does
    not change the device default pool's release threshold."""
    import ctypes

    cudart = None
    for name in ("libcudart.so.12", "libcudart.so"):
        try:
            cudart = ctypes.CDLL(name)
            break
        except OSError:
            continue
    if cudart is None:
        pytest.skip("libcudart not loadable by name")
    pool = ctypes.c_void_p()
    assert cudart.cudaDeviceGetDefaultMemPool(ctypes.byref(pool), 0) == 0
    before = ctypes.c_uint64()
    assert cudart.cudaMemPoolGetAttribute(pool, 4, ctypes.byref(before)) == 0  # ReleaseThreshold
    params = B.BfvParams(B.RnsContext(128, PRIMES), 257)
    g = E.GpuContext(params)
    del g
    after = ctypes.c_uint64()
    assert cudart.cudaMemPoolGetAttribute(pool, 4, ctypes.byref(after)) == 0
    assert after.value == before.value
