#!/usr/bin/env python3
"""Generate the golden vectors of the hot path FROM THE REFERENCE ITSELF.

Runs only in the build container, where the reference (`hefir`) is mounted
read-only at /root/reference/pkg/src.  gmpy2 is absent there, so a one-line
shim (`tests/_shim/gmpy2.py`: `mpz = int`) is put on the path; it yields the
same exact integers (the reference uses gmpy2 only for one big-int multiply,
ring.py:324-326).

Outputs (committed; small):
  small.npz / small.json       N=64, 4 pool primes, t=257: NTT KAT, hmult_raw,
                               relinearize, hsquare on random and edge-value
                               ciphertexts, conv/pool/fc layers, toy network.
  n1024.npz / n1024.json       N=1024, the 11 set-1 primes, MNIST t: hsquare on
                               random and edge-value ciphertexts.
  cifar64.npz / cifar64.json   N=64, CIFAR t_0: padded conv + pool + square.
  mnist1024.json (+ mnist_fixture_weights.npz)
                               The MNIST HCNN on the reference's 4-bit fixture
                               model at N=1024 / set-1 primes: per-layer
                               sha256 digests, op counters, decrypted logits.
  set1.json                    N=8192 set 1: digests of keys, one ciphertext,
                               its hmult_raw and hsquare (full-size pin).
  set1net.json / set1net.npz   The bench workload itself (bench.py, seed 2024):
                               MNIST HCNN at set 1, dense random 4-bit weights,
                               one 8192-image slot-batch, evaluated by the
                               reference's eval_network; every layer's sha256
                               (all limbs of all ciphertexts), the counters and
                               the decrypted logits of all 8192 images.
  plain.npz / plain.json       hmult_plain, scalar and NTT paths, 2- and 3-part
                               ciphertexts (N=64 arrays, N=1024 digests).
  hfir.npz / hfir.json         HFIR bytes of a cipher tensor, a 3-part
                               ciphertext and a relinearisation key.

Usage: python tests/golden/make_golden.py [small n1024 cifar64 mnist1024 set1 plain hfir set1net]
(set1net is not in the default list: ~25 minutes on 8 cores.)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [os.path.join(REPO, "tests", "_shim"), "/root/reference/pkg/src"]
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")

import numpy as np  # noqa: E402

from hefir import bfv, engine, nn_oracle, presets, ring, serial  # noqa: E402
from hefir.batching import SlotEncoder  # noqa: E402

POOL = presets.RNS_PRIME_POOL
MNIST_T = presets.MNIST_T
CIFAR_T = presets.CIFAR_T


def u32(arr):
    return np.asarray(arr, dtype=np.int64).astype(np.uint32)


def ct_arr(c):
    return np.stack([p.residues for p in c.parts])


def digest_cts(cts) -> str:
    h = hashlib.sha256()
    for c in cts:
        for part in c.parts:
            h.update(np.ascontiguousarray(part.residues.astype("<u8")).tobytes())
    return h.hexdigest()


def counter_dict(c):
    return dict(
        mult_plain_scheduled=c.mult_plain_scheduled,
        mult_plain_executed=c.mult_plain_executed,
        mult_plain_skipped=c.mult_plain_skipped,
        hsquare=c.hsquare,
        hadd=c.hadd,
    )


def rlk_arr(rlk):
    return np.stack([np.stack([k0.residues, k1.residues]) for k0, k1 in rlk.components])


def edge_cts(params, rng):
    """Ciphertexts whose canonical lifts sit at 0, 1, q-1 and near q.

    These stress exact base conversion: a floating-point CRT overflow
    estimate is ambiguous exactly when the lifted value is near 0 or q.
    """
    ctx = params.ctx
    q = ctx.q_big
    n = ctx.ring_degree

    def from_ints(vals):
        return ring.crt_reduce(ring.BigPoly.from_ints([v % q for v in vals]), ctx)

    zero = [0] * n
    minus1 = [q - 1] * n
    mixed = []
    for j in range(n):
        sel = j % 6
        if sel == 0:
            mixed.append(int(rng.integers(0, 40)))
        elif sel == 1:
            mixed.append(q - 1 - int(rng.integers(0, 40)))
        elif sel == 2:
            mixed.append(q - (1 << int(rng.integers(1, q.bit_length() - 30))))
        elif sel == 3:
            mixed.append((1 << int(rng.integers(1, q.bit_length() - 1))))
        elif sel == 4:
            mixed.append(q // 2 + int(rng.integers(-3, 4)))
        else:
            mixed.append(int.from_bytes(rng.bytes(64), "little") % q)
    out = []
    for a, b in ((zero, zero), (minus1, minus1), (mixed, list(reversed(mixed))), (zero, minus1)):
        out.append(bfv.Ciphertext(parts=(from_ints(a), from_ints(b)), fingerprint=params.fingerprint))
    return out


def make_small():
    ctx = ring.RnsContext(64, list(POOL[:4]))
    params = bfv.BfvParams(ctx, 257)
    sk, pk, rlk = bfv.keygen(params, np.random.default_rng(101))
    rng = np.random.default_rng(7)
    x = np.stack([rng.integers(0, p, 64) for p in POOL[:4]])
    xf = ring.ntt_forward(ring.RingElem(ctx, x.copy(), ring.Domain.COEFF)).residues
    erng = np.random.default_rng(11)
    cts = [
        bfv.encrypt(pk, bfv.Plaintext(erng.integers(0, 257, 64), 257), params, erng)
        for _ in range(3)
    ] + edge_cts(params, np.random.default_rng(12))
    raw = [bfv.hmult_raw(c, c, params) for c in cts]
    hsq = [bfv.hsquare(c, rlk, params) for c in cts]
    gen = bfv.hmult_raw(cts[0], cts[1], params)
    gen_rl = bfv.hmult(cts[0], cts[1], rlk, params)

    # layer-level: a (5,5,2) tensor through padded/grouped/strided convs, pool, fc
    lrng = np.random.default_rng(21)
    tens_cts = [
        bfv.encrypt(pk, bfv.Plaintext(lrng.integers(0, 257, 64), 257), params, lrng)
        for _ in range(5 * 5 * 2)
    ]
    tensor = engine.CipherTensor(shape=(5, 5, 2), cts=tens_cts, delta=4, channel_modulus=257)
    layers = {}
    cnt = {}
    cases = [
        ("conv_pad_s1", nn_oracle.conv_layer("c", 4, (3, 3), (1, 1), True, 15)),
        ("conv_s2_g2", nn_oracle.conv_layer("c", 4, (3, 3), (2, 2), False, 15, groups=2)),
        ("conv_pad_s2_g2", nn_oracle.conv_layer("c", 2, (3, 3), (2, 2), True, 15, groups=2)),
    ]
    for name, layer in cases:
        cg = 2 // layer.groups
        w = lrng.integers(-4, 5, (layer.filters, 3, 3, cg))
        w[0, 0, 0, 0] = 0
        if name == "conv_s2_g2":
            w[1] = 0  # a filter with no executed taps -> zero ciphertext
        counter = engine.OpCounter()
        out = engine.eval_conv(tensor, layer, w, params, counter)
        layers[name + "_w"] = w
        layers[name + "_out"] = u32([ct_arr(c) for c in out.cts])
        cnt[name] = counter_dict(counter)
        cnt[name]["shape"] = list(out.shape)
    counter = engine.OpCounter()
    pl = nn_oracle.pool_layer("p", 2, 2)
    out = engine.eval_pool(tensor, pl, params, counter)
    layers["pool_out"] = u32([ct_arr(c) for c in out.cts])
    cnt["pool"] = counter_dict(counter)
    cnt["pool"]["shape"] = list(out.shape)
    fw = lrng.integers(-1000, 1000, (3, 50))
    fw[1, ::3] = 0
    fw[2, 5] = 2**40 + 3  # large weight: w mod p path
    fw[0, 7] = -(2**35)
    counter = engine.OpCounter()
    out = engine.eval_fc(tensor, nn_oracle.fc_layer("f", 3, 15), fw, params, counter)
    layers["fc_w"] = fw
    layers["fc_out"] = u32([ct_arr(c) for c in out.cts])
    cnt["fc"] = counter_dict(counter)

    # toy network end to end (engine.py:400-423) on 5 packed 8x8 images
    spec = nn_oracle.toy_hcnn()
    wrng = np.random.default_rng(31)
    weights = [wrng.integers(-4, 5, (2, 3, 3, 1)), None, wrng.integers(-4, 5, (3, 18))]
    model = nn_oracle.QuantizedModel(spec=spec, bit_width=4, weights=weights)
    enc = SlotEncoder(257, 64)
    images = [np.random.default_rng(41 + i).integers(0, 5, (8, 8, 1)) for i in range(5)]
    prng = np.random.default_rng(51)
    layout = engine.PackingLayout(5, 64)
    tin = engine.pack_images(images, layout, enc, pk, params, prng, delta=4)
    hooks = {}

    def hook(name, t):
        hooks[name] = u32([ct_arr(c) for c in t.cts])

    counter = engine.OpCounter()
    tout = engine.eval_network(tin, model, rlk, params, counter, layer_hook=hook)
    vals = engine.unpack_tensor(tout, sk, enc, params, 5)
    plain = [nn_oracle.forward(model, im).reshape(-1) for im in images]

    np.savez_compressed(
        os.path.join(HERE, "small.npz"),
        rlk=u32(rlk_arr(rlk)),
        pk=u32(np.stack([pk.b_ntt.residues, pk.a_ntt.residues])),
        s_bits=sk.s_bits.astype(np.uint8),
        ntt_in=u32(x),
        ntt_out=u32(xf),
        cts=u32([ct_arr(c) for c in cts]),
        raw=u32([ct_arr(c) for c in raw]),
        hsq=u32([ct_arr(c) for c in hsq]),
        gen_raw=u32(ct_arr(gen)),
        gen_hmult=u32(ct_arr(gen_rl)),
        tensor_in=u32([ct_arr(c) for c in tens_cts]),
        toy_in=u32([ct_arr(c) for c in tin.cts]),
        toy_conv1=hooks["conv1"],
        toy_square1=hooks["square1"],
        toy_fc=hooks["fc"],
        toy_w_conv1=weights[0],
        toy_w_fc=weights[2],
        toy_images=np.stack(images),
        toy_decrypted=vals,
        toy_plain=np.stack(plain).astype(np.int64),
        **layers,
    )
    meta = dict(
        n=64, primes=list(POOL[:4]), t=257, keys_seed=101,
        counters=cnt, toy_counter=counter_dict(counter),
        toy_delta=tout.delta,
        digests=dict(
            hsq=digest_cts(hsq),
            toy_in=digest_cts(tin.cts),
        ),
    )
    with open(os.path.join(HERE, "small.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def make_n1024():
    ctx = ring.RnsContext(1024, list(POOL[:11]))
    params = bfv.BfvParams(ctx, MNIST_T)
    sk, pk, rlk = bfv.keygen(params, np.random.default_rng(202))
    erng = np.random.default_rng(13)
    cts = [
        bfv.encrypt(pk, bfv.Plaintext(erng.integers(0, MNIST_T, 1024), MNIST_T), params, erng)
        for _ in range(2)
    ] + edge_cts(params, np.random.default_rng(14))[1:3]
    t0 = time.time()
    raw0 = bfv.hmult_raw(cts[0], cts[0], params)
    hsq = [bfv.hsquare(c, rlk, params) for c in cts]
    print(f"n1024 hsquare x{len(cts)}: {time.time() - t0:.1f}s")
    np.savez_compressed(
        os.path.join(HERE, "n1024.npz"),
        cts=u32([ct_arr(c) for c in cts]),
        raw0=u32(ct_arr(raw0)),
        hsq=u32([ct_arr(c) for c in hsq]),
    )
    meta = dict(
        n=1024, primes=list(POOL[:11]), t=MNIST_T, keys_seed=202,
        digests=dict(rlk=hashlib.sha256(rlk_arr(rlk).astype("<u8").tobytes()).hexdigest(),
                     hsq=digest_cts(hsq)),
    )
    with open(os.path.join(HERE, "n1024.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def make_cifar64():
    t = CIFAR_T[0]
    ctx = ring.RnsContext(64, list(POOL[:10]))
    params = bfv.BfvParams(ctx, t)
    sk, pk, rlk = bfv.keygen(params, np.random.default_rng(808))
    enc = SlotEncoder(t, 64)
    images = [np.random.default_rng(60 + i).integers(0, 256, (4, 4, 3)) for i in range(3)]
    prng = np.random.default_rng(61)
    tin = engine.pack_images(images, engine.PackingLayout(3, 64), enc, pk, params, prng, delta=255)
    wrng = np.random.default_rng(62)
    w = wrng.integers(-20, 21, (4, 3, 3, 3))
    conv = nn_oracle.conv_layer("conv", 4, (3, 3), (1, 1), True, 10000)
    pool = nn_oracle.pool_layer("pool", 2, 2)
    counter = engine.OpCounter()
    a = engine.eval_conv(tin, conv, w, params, counter)
    b = engine.eval_square(a, rlk, params, counter)
    c = engine.eval_pool(b, pool, params, counter)
    vals = engine.unpack_tensor(c, sk, enc, params, 3)
    np.savez_compressed(
        os.path.join(HERE, "cifar64.npz"),
        tin=u32([ct_arr(x) for x in tin.cts]),
        w=w,
        conv=u32([ct_arr(x) for x in a.cts]),
        square=u32([ct_arr(x) for x in b.cts]),
        pool=u32([ct_arr(x) for x in c.cts]),
        decrypted=vals,
        images=np.stack(images),
    )
    meta = dict(n=64, primes=list(POOL[:10]), t=t, keys_seed=808, counter=counter_dict(counter),
                shapes=[list(a.shape), list(b.shape), list(c.shape)])
    with open(os.path.join(HERE, "cifar64.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def make_mnist1024():
    ctx = ring.RnsContext(1024, list(POOL[:11]))
    params = bfv.BfvParams(ctx, MNIST_T)
    sk, pk, rlk = bfv.keygen(params, np.random.default_rng(303))
    with open("/root/reference/pkg/data/models/mnist_fixture_4bit.json") as fh:
        model = serial.load_model(fh.read())
    np.savez_compressed(
        os.path.join(HERE, "mnist_fixture_weights.npz"),
        conv1=model.weights[0], conv2=model.weights[2], fc=model.weights[4],
    )
    batch = 16
    irng = np.random.default_rng(404)
    images = [irng.integers(0, 5, (28, 28, 1)) for _ in range(batch)]
    enc = SlotEncoder(MNIST_T, 1024)
    prng = np.random.default_rng(505)
    t0 = time.time()
    tin = engine.pack_images(images, engine.PackingLayout(batch, 1024), enc, pk, params, prng, delta=4)
    print(f"mnist1024 pack: {time.time() - t0:.1f}s")
    digests = {"input": digest_cts(tin.cts)}
    times = {}
    last = [time.time()]

    def hook(name, t):
        digests[name] = digest_cts(t.cts)
        times[name] = time.time() - last[0]
        last[0] = time.time()
        print(f"  {name}: {times[name]:.1f}s", flush=True)

    counter = engine.OpCounter()
    tout = engine.eval_network(tin, engine.reduce_model(model, MNIST_T), rlk, params, counter,
                               workers=8, layer_hook=hook)
    vals = engine.unpack_tensor(tout, sk, enc, params, batch)
    plain = [nn_oracle.forward(model, im).reshape(-1) for im in images]
    meta = dict(
        n=1024, primes=list(POOL[:11]), t=MNIST_T, keys_seed=303, image_seed=404,
        image_count=batch, pack_seed=505, digests=digests, counter=counter_dict(counter),
        delta=tout.delta, decrypted=vals.tolist(), plain=[[int(v) for v in p] for p in plain],
        labels=[nn_oracle.classify(p) for p in plain], layer_seconds=times,
    )
    with open(os.path.join(HERE, "mnist1024.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def make_set1():
    p = presets.load_preset("1")
    params = presets.build_context(p)
    sk, pk, rlk = bfv.keygen(params, np.random.default_rng(606))
    erng = np.random.default_rng(707)
    c = bfv.encrypt(pk, bfv.Plaintext(erng.integers(0, MNIST_T, 8192), MNIST_T), params, erng)
    t0 = time.time()
    raw = bfv.hmult_raw(c, c, params)
    t1 = time.time()
    h = bfv.hsquare(c, rlk, params)
    t2 = time.time()
    meta = dict(
        n=8192, primes=list(p.rns_primes), t=MNIST_T, keys_seed=606, enc_seed=707,
        digests=dict(
            rlk=hashlib.sha256(rlk_arr(rlk).astype("<u8").tobytes()).hexdigest(),
            ct=digest_cts([c]), raw=digest_cts([raw]), hsq=digest_cts([h]),
        ),
        seconds=dict(hmult_raw=t1 - t0, hsquare=t2 - t1),
    )
    with open(os.path.join(HERE, "set1.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


_SQ = {}


def _sq_worker(i):
    return bfv.hsquare(_SQ["cts"][i], _SQ["rlk"], _SQ["params"])


def _pool_eval_square(tensor, rlk, params, counter, workers=1):
    """engine.eval_square (engine.py:337-364) with the per-ciphertext
    bfv.hsquare calls fanned over forked processes instead of GIL-bound
    threads: same calls, same outputs, same counter and delta updates."""
    import multiprocessing as mp

    _SQ.update(cts=tensor.cts, rlk=rlk, params=params)
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        out = pool.map(_sq_worker, range(len(tensor.cts)), chunksize=1)
    counter.hsquare += len(out)
    return engine.CipherTensor(shape=tensor.shape, cts=out, delta=tensor.delta * tensor.delta,
                               channel_modulus=tensor.channel_modulus)


def make_set1net(seed: int = 2024):
    """bench.py's MNIST step (build_workload, seed 2024) run by the reference.

    Same derivations as bench.build_workload: weights nn.random_model(spec,
    default_rng(seed+1)), keys bfv.keygen(default_rng(seed)), images
    default_rng(seed+100).integers(0, 5, (8192, 28, 28, 1)), packing rng
    default_rng(seed+200), delta 4."""
    sys.path.insert(0, REPO)
    from paper_1811_00778_b200 import nn as mynn

    p = presets.load_preset("1")
    params = presets.build_context(p)
    n = params.ring_degree
    spec = nn_oracle.mnist_hcnn()
    mine = mynn.random_model(mynn.mnist_hcnn(), np.random.default_rng(seed + 1))
    model = nn_oracle.QuantizedModel(spec=spec, bit_width=4, weights=mine.weights)
    t0 = time.time()
    sk, pk, rlk = bfv.keygen(params, np.random.default_rng(seed))
    images = list(np.random.default_rng(seed + 100).integers(0, 5, (n, 28, 28, 1)))
    enc = SlotEncoder(MNIST_T, n)
    tin = engine.pack_images(images, engine.PackingLayout(n, n), enc, pk, params,
                             np.random.default_rng(seed + 200), delta=4)
    print(f"set1net keys+pack: {time.time() - t0:.1f}s", flush=True)
    digests = {"input": digest_cts(tin.cts)}
    times = {}
    last = [time.time()]

    def hook(name, t):
        digests[name] = digest_cts(t.cts)
        times[name] = time.time() - last[0]
        last[0] = time.time()
        print(f"  {name}: {times[name]:.1f}s {digests[name][:16]}", flush=True)

    counter = engine.OpCounter()
    engine.eval_square = _pool_eval_square  # eval_network resolves it at call time
    tout = engine.eval_network(tin, engine.reduce_model(model, MNIST_T), rlk, params, counter,
                               workers=8, layer_hook=hook)
    vals = engine.unpack_tensor(tout, sk, enc, params, n)  # (batch, 10) in [0, t)
    np.savez_compressed(os.path.join(HERE, "set1net.npz"), decrypted=vals.astype(np.int64))
    meta = dict(
        n=n, primes=list(p.rns_primes), t=MNIST_T, seed=seed, keys_seed=seed, image_seed=seed + 100,
        pack_seed=seed + 200, weights_seed=seed + 1, digests=digests, counter=counter_dict(counter),
        delta=tout.delta, layer_seconds=times, cpu_count=os.cpu_count(),
        rlk=hashlib.sha256(rlk_arr(rlk).astype("<u8").tobytes()).hexdigest(),
        logits_sha=hashlib.sha256(vals.astype("<i8").tobytes()).hexdigest(),
        note="square layers: bfv.hsquare per ciphertext over a fork pool (same calls as engine.eval_square)",
    )
    with open(os.path.join(HERE, "set1net.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def make_plain():
    """hmult_plain (bfv.py:301-318): NTT path (random, sparse, high-degree
    plaintexts) and scalar path (constants, both signs), 2- and 3-part
    ciphertexts, at N=64 (t=257) and N=1024 with the set-1 primes."""
    arrays, meta = {}, {}
    for tag, n, k, t, seed in (("s", 64, 4, 257, 111), ("m", 1024, 11, MNIST_T, 222)):
        ctx = ring.RnsContext(n, list(POOL[:k]))
        params = bfv.BfvParams(ctx, t)
        sk, pk, rlk = bfv.keygen(params, np.random.default_rng(seed))
        rng = np.random.default_rng(seed + 1)
        cts = [bfv.encrypt(pk, bfv.Plaintext(rng.integers(0, t, n), t), params, rng) for _ in range(2)]
        cts += edge_cts(params, np.random.default_rng(seed + 2))[1:3]
        pts = [rng.integers(0, t, n)]
        sparse = np.zeros(n, dtype=np.int64)
        sparse[[1, n - 1]] = [t - 1, 3]
        pts.append(sparse)
        top = np.zeros(n, dtype=np.int64)
        top[n - 1] = t // 2 + 1
        pts.append(top)
        for v in (200 % t, t - 5, 7, 0):
            pts.append(bfv.Plaintext.constant(v, params).poly)
        outs = np.stack([np.stack([ct_arr(bfv.hmult_plain(c, bfv.Plaintext(pt, t), params)) for c in cts])
                         for pt in pts])
        raw3 = bfv.hmult_raw(cts[0], cts[1], params)
        out3 = [ct_arr(bfv.hmult_plain(raw3, bfv.Plaintext(pt, t), params)) for pt in pts[:2]]
        arrays.update({
            f"{tag}_cts": u32([ct_arr(c) for c in cts]),
            f"{tag}_pts": np.stack(pts).astype(np.int64),
            f"{tag}_raw3": u32(ct_arr(raw3)),
        })
        meta[tag] = dict(n=n, primes=list(POOL[:k]), t=t)
        if tag == "s":  # full outputs at N=64, sha256 of the u64 LE residues at N=1024
            arrays.update({f"{tag}_out": u32(outs), f"{tag}_out3": u32(out3)})
        else:
            meta[tag]["out_sha"] = [hashlib.sha256(o.astype("<u8").tobytes()).hexdigest() for o in outs]
            meta[tag]["out3_sha"] = [hashlib.sha256(np.asarray(o).astype("<u8").tobytes()).hexdigest()
                                     for o in out3]
    np.savez_compressed(os.path.join(HERE, "plain.npz"), **arrays)
    with open(os.path.join(HERE, "plain.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def make_hfir():
    """HFIR bytes (serial.py:44-229) of a cipher tensor with fresh and
    evaluated ciphertexts, a 3-part ciphertext and a relinearisation key:
    the byte-exact target of the device-side HFIR reader/writer."""
    ctx = ring.RnsContext(64, list(POOL[:4]))
    params = bfv.BfvParams(ctx, 257)
    sk, pk, rlk = bfv.keygen(params, np.random.default_rng(121))
    rng = np.random.default_rng(122)
    cts = [bfv.encrypt(pk, bfv.Plaintext(rng.integers(0, 257, 64), 257), params, rng) for _ in range(5)]
    cts[3] = bfv.hsquare(cts[3], rlk, params)  # is_fresh False
    tensor = engine.CipherTensor(shape=(1, 5, 1), cts=cts, delta=3 * 2**70 + 5, channel_modulus=257)
    blob = serial.dump_cipher_tensor(tensor, params)
    raw3 = bfv.hmult_raw(cts[0], cts[1], params)
    np.savez_compressed(
        os.path.join(HERE, "hfir.npz"),
        tensor=np.frombuffer(blob, dtype=np.uint8),
        cts=u32([ct_arr(c) for c in cts]),
        fresh=np.array([c.is_fresh for c in cts]),
        ct3=np.frombuffer(serial.dump_ciphertext(raw3, params), dtype=np.uint8),
        raw3=u32(ct_arr(raw3)),
        rlk_file=np.frombuffer(serial.dump_relin_key(rlk, params), dtype=np.uint8),
        rlk=u32(rlk_arr(rlk)),
    )
    meta = dict(n=64, primes=list(POOL[:4]), t=257, keys_seed=121, delta=tensor.delta, shape=[1, 5, 1])
    with open(os.path.join(HERE, "hfir.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def make_ntt64():
    """u64 NTT known answers through the reference's own tables and transform
    (ntt.NttPlan: psi search, twists, stage-packed twiddles;
    ntt._transform_rows_numpy on Python ints, exact for 62-bit primes;
    ring.ntt_forward / ntt_inverse's twist and untwist): natural-order
    spectra of seeded rows for a 62-bit prime and for the MNIST t."""
    from hefir import ntt as _ntt

    def prime_below(bits, two_n):
        k = ((1 << bits) - 1) // two_n
        while True:
            cand = k * two_n + 1
            if cand < (1 << bits) and _ntt.is_probable_prime(cand):
                return cand
            k -= 1

    p62 = prime_below(62, 1 << 16)
    rng = np.random.default_rng(64)
    out, meta = {}, {"p62": p62, "cases": []}
    for name, p, n in (("p62_64", p62, 64), ("p62_1024", p62, 1024), ("p62_8192", p62, 8192),
                       ("t_8192", MNIST_T, 8192)):
        plan = _ntt.NttPlan(p, n)
        rev = _ntt.bit_reverse_indices(n)
        x = np.array([[int(v) for v in rng.integers(0, p, n, dtype=np.uint64)] for _ in range(2)], dtype=object)
        x[1, :8] = p - 1
        mods = np.array([p, p], dtype=object)
        tw = np.array([plan.tw, plan.tw], dtype=object)
        itw = np.array([plan.itw, plan.itw], dtype=object)
        fwd = x * np.array(plan.psi_pows, dtype=object) % p          # ring.ntt_forward: twist,
        _ntt._transform_rows_numpy(fwd, mods, tw, rev)                # then the cyclic transform
        inv = x.copy()                                                # ring.ntt_inverse of x
        _ntt._transform_rows_numpy(inv, mods, itw, rev)
        inv = inv * np.array(plan.ipsi_pows, dtype=object) % p
        out[name + "_x"] = x.astype(np.uint64)
        out[name + "_fwd"] = fwd.astype(np.uint64)
        out[name + "_inv"] = inv.astype(np.uint64)
        meta["cases"].append({"name": name, "p": p, "n": n})
    np.savez_compressed(os.path.join(HERE, "ntt64.npz"), **out)
    with open(os.path.join(HERE, "ntt64.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "n1024", "cifar64", "set1", "mnist1024", "plain", "hfir"]
    for w in which:
        t0 = time.time()
        globals()["make_" + w]()
        print(f"{w}: {time.time() - t0:.1f}s", flush=True)
