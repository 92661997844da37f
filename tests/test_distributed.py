"""Multi-process (world size 2, gloo on CPU) checks of the sharding plan, the
final gather and the CRT recombination used by the multi-GPU path."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_00778_b200 import distributed as D
from paper_1811_00778_b200 import engine as E


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        moduli = (257, 65537, 2424833)
        n_batches = 3
        plan = D.shard_plan(n_batches, len(moduli), world)
        signed = {b: np.arange(-6, 6).reshape(3, 4) * (b + 1) * 1000 for b in range(n_batches)}

        def evaluate(u):
            # stand-in for a homomorphic evaluation: the "logit ciphertext"
            # carries the signed logits reduced mod this unit's channel modulus
            t = moduli[u.channel]
            return torch.from_numpy((signed[u.batch] % t).astype(np.int64))

        res = D.run_units(evaluate, plan, rank, world)
        if rank == 0:
            assert set(res) == {D.Unit(b, c) for b in range(n_batches) for c in range(len(moduli))}
            logits = D.recombine(res, lambda u, t: t.numpy(), moduli, n_batches)
            ok = all(np.array_equal(logits[b].astype(np.int64), signed[b].T) for b in range(n_batches))
            q.put(ok)
    finally:
        dist.destroy_process_group()


def test_plan_covers_units_once():
    for world in (1, 2, 3, 8):
        plan = D.shard_plan(4, 10, world)
        flat = [u for p in plan for u in p]
        assert len(flat) == 40 and len(set(flat)) == 40
        assert max(len(p) for p in plan) - min(len(p) for p in plan) <= 1


def test_gather_and_recombine_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def test_reconstruct_matches_reference_formula():
    moduli = (2424833, 2654209, 2752513)
    res = E.ChannelResult(moduli=moduli, batch_size=2)
    vals = np.array([[123456789012, -98765432100], [-1, 0]], dtype=object)
    for t in moduli:
        res.add(t, np.vectorize(lambda v: int(v) % t)(vals).astype(np.int64))
    got = E.reconstruct_logits(res, moduli)
    assert (got == vals.T).all()
    _ = pytest


# ------------------------------------------------------------------ output-channel groups


def _mnist_like(rng, n=64):
    """MNIST-shaped grouped network at a small ring: 12x12 input, conv 3@3x3
    s1, square, conv 6@3x3 s2 groups 3, square, fc 4."""
    import hcnn_oracle as O  # noqa: F401

    from paper_1811_00778_b200 import nn

    spec = nn.NetworkSpec("mini", (12, 12, 1), 4, (
        nn.conv_layer("conv1", 3, (3, 3), (1, 1), False, 15),
        nn.square_layer_spec("square1"),
        nn.conv_layer("conv2", 6, (3, 3), (2, 2), False, 15, groups=3),
        nn.square_layer_spec("square2"),
        nn.fc_layer("fc", 4, 15),
    ))
    w = [rng.integers(-3, 4, (3, 3, 3, 1)), None, rng.integers(-3, 4, (6, 3, 3, 1)), None,
         rng.integers(-3, 4, (4, 4 * 4 * 6))]
    return nn.QuantizedModel(spec, 4, w)


def _layers(model):
    out = []
    for layer, w in zip(model.spec.layers, model.weights):
        k = layer.kind.value
        d = {"kind": k, "name": layer.name}
        if k == "conv":
            d.update(kernel=layer.kernel, stride=layer.stride, padded=layer.padded, groups=layer.groups,
                     weight_scale=layer.weight_scale, weights=w)
        elif k == "fc":
            d.update(weight_scale=layer.weight_scale, weights=w)
        out.append(d)
    return out


def test_group_slices_sum_to_the_full_network():
    """Per-group sub-networks (plaintext integer network) sum to the full
    network's logits for every world size, and the group plan covers every
    group once."""
    import hcnn_oracle as O

    rng = np.random.default_rng(8)
    model = _mnist_like(rng)
    assert D.groupable(model.spec) == 3
    image = rng.integers(0, 5, (12, 12, 1))
    full = O.plain_forward(_layers(model), image).reshape(-1)
    for world in (1, 2, 3, 5):
        plan = D.group_plan(3, world)
        assert sorted(g for p in plan for g in p) == [0, 1, 2]
        total = sum(O.plain_forward(_layers(D.slice_model(model, sel)), image).reshape(-1)
                    for sel in plan if sel)
        assert [int(v) for v in total] == [int(v) for v in full]
    assert D.output_delta(model.spec, 4) == ((4 * 15) ** 2 * 15) ** 2 * 15


def _group_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import hcnn_oracle as O

        rng = np.random.default_rng(8)
        model = _mnist_like(rng)
        image = rng.integers(0, 5, (12, 12, 1))
        p = 65537
        sel = D.group_plan(3, world)[rank]
        part = O.plain_forward(_layers(D.slice_model(model, sel)), image).reshape(-1) if sel else np.zeros(4)
        send = torch.tensor([int(v) % p for v in part], dtype=torch.int64)
        bufs = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
        dist.gather(send, bufs, dst=0)
        if rank == 0:
            got = sum(b for b in bufs) % p
            full = O.plain_forward(_layers(model), image).reshape(-1)
            q.put([int(v) for v in got] == [int(v) % p for v in full])
    finally:
        dist.destroy_process_group()


def test_group_partials_gather_world2():
    """The partial logits of two ranks, gathered with gloo and added mod p,
    equal the full network's logits mod p (the collective of
    distributed.eval_network_groups)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_group_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    ok = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
    assert ok
