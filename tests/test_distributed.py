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


# ---------------------------------------------------------------- CRT channels + output-channel split


def test_channel_plan_balances_cifar_on_1_2_4_8_ranks():
    for world, per_rank in ((1, 10), (2, 5), (4, 2.5), (8, 1.25), (3, 10 / 3)):
        whole, splits = D.channel_plan(10, world)
        load = [len(w) for w in whole]
        covered = [c for w in whole for c in w] + [c for c, _ in splits]
        assert sorted(covered) == list(range(10))
        for c, ranks in splits:
            for r in ranks:
                load[r] += 1 / len(ranks)
        assert max(load) == pytest.approx(per_rank), (world, load)
    whole, splits = D.channel_plan(10, 8)
    assert whole == [[r] for r in range(8)] and splits == [(8, [0, 1, 2, 3]), (9, [4, 5, 6, 7])]


class _OTensor:
    """CPU stand-in for a GpuCipherTensor: int64 [n][2][K][N] residues."""

    def __init__(self, shape, data, delta):
        self.shape, self.data, self.delta = tuple(shape), data, delta

    def __len__(self):
        return self.data.shape[0]


class _OracleBackend:
    """The split program's layer operations on the pinned oracle (CPU)."""

    def __init__(self, op, rlk):
        self.op, self.rlk = op, rlk

    def _ot(self, x):
        import hcnn_oracle as O

        d = x.data.numpy()
        return O.Tensor(x.shape, [(c[0], c[1]) for c in d], x.delta)

    def _back(self, ot):
        return _OTensor(ot.shape, torch.from_numpy(np.stack([np.stack(c) for c in ot.cts]).astype(np.int64)),
                        ot.delta)

    def conv(self, x, layer, w, counter):
        import hcnn_oracle as O

        return self._back(O.conv(self.op, self._ot(x), layer.kernel, layer.stride, layer.padded, layer.groups,
                                 layer.weight_scale, w, counter))

    def square(self, x, counter):
        import hcnn_oracle as O

        return self._back(O.square(self.op, self._ot(x), self.rlk, counter))

    def pool(self, x, layer, counter):
        import hcnn_oracle as O

        return self._back(O.pool(self.op, self._ot(x), layer.extent, layer.stride, counter))

    def fc(self, x, layer, w, counter):
        import hcnn_oracle as O

        return self._back(O.fc(self.op, self._ot(x), w, layer.weight_scale, counter))

    def wrap(self, shape, data, delta):
        return _OTensor(shape, data, delta)

    def add(self, a, b):
        mods = torch.from_numpy(self.op.ctx.mods.reshape(1, 1, -1, 1))
        return (a + b) % mods


def _split_world():
    """Tiny CIFAR-shaped network (padded dense convs, squares, pools, two
    dense layers) at N=64 with 4 pool primes, t = 257, and its inputs."""
    import hcnn_oracle as O

    from paper_1811_00778_b200 import nn

    n, primes, t = 64, [1073643521, 1073479681, 1073184769, 1073053697], 257
    op = O.Params(O.Context(n, primes), t)
    rng = np.random.default_rng(90)
    _, _, rlk = O.keygen(op, rng)
    spec = nn.NetworkSpec("mini_cifar", (6, 6, 2), 255, (
        nn.conv_layer("conv1", 5, (3, 3), (1, 1), True, 10),
        nn.square_layer_spec("square1"),
        nn.pool_layer("pool1", 2, 2),
        nn.conv_layer("conv2", 7, (3, 3), (1, 1), True, 10),
        nn.square_layer_spec("square2"),
        nn.pool_layer("pool2", 2, 1),
        nn.fc_layer("fc1", 4, 5),
        nn.fc_layer("fc2", 3, 5),
    ))
    model = nn.random_model(spec, np.random.default_rng(91))
    mods = op.ctx.mods.reshape(1, 1, -1, 1)
    x = np.random.default_rng(92).integers(0, 1 << 30, (72, 2, 4, n)) % mods
    return op, rlk, model, x


def _full_network(op, rlk, model, x):
    import hcnn_oracle as O
    from helpers import layer_dicts

    c = O.Counter()
    out = O.network(op, O.Tensor((6, 6, 2), [(d[0], d[1]) for d in x], 255), layer_dicts(model.spec, model.weights),
                    rlk, c)
    return np.stack([np.stack(ct) for ct in out.cts]), c


def test_split_program_emulated_equals_the_full_network():
    """All S ranks of one channel's output-channel split run in lockstep in
    one process (the single-GPU emulation driver), on the oracle: the
    reassembled logits equal the unsplit network bit for bit, and the ranks'
    counters add up to the unsplit counter."""
    import hcnn_oracle as O

    op, rlk, model, x = _split_world()
    exp, ec = _full_network(op, rlk, model, x)
    be = _OracleBackend(op, rlk)
    for S in (2, 3):
        counters = [O.Counter() for _ in range(S)]
        out = D.run_split_emulated(_OTensor((6, 6, 2), torch.from_numpy(x), 255), model, be, S, counters)
        assert np.array_equal(out.data.numpy(), exp), S
        tot = {k: sum(getattr(c, k) for c in counters) for k in ec.__dict__}
        assert tot == ec.__dict__, S


def _split_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import hcnn_oracle as O

        op, rlk, model, x = _split_world()
        c = O.Counter()
        out = D.run_split(_OTensor((6, 6, 2), torch.from_numpy(x), 255), model, _OracleBackend(op, rlk),
                          list(range(world)), rank, None, c)
        cs = [None] * world
        dist.all_gather_object(cs, c.__dict__)
        if rank == 0:
            exp, ec = _full_network(op, rlk, model, x)
            tot = {k: sum(d[k] for d in cs) for k in ec.__dict__}
            q.put(bool(np.array_equal(out.data.numpy(), exp)) and tot == ec.__dict__)
        else:
            assert out is None
    finally:
        dist.destroy_process_group()


def test_split_program_over_two_gloo_ranks():
    """The same split with real torch.distributed collectives (gloo, world
    size 2): all-gather of the channel slices before conv2, gather of the fc
    partial sums to rank 0."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def _recombine_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        moduli = (2424833, 2654209, 2752513, 2819073)
        signed = np.array([[123456789012345, -9876543210987], [-1, 0], [5, -5]], dtype=object)  # (outputs, batch)
        owners = {D.Unit(0, c): c % world for c in range(len(moduli))}
        local = {u: torch.from_numpy(np.vectorize(lambda v, t=moduli[u.channel]: int(v) % t)(signed).astype(np.int64))
                 for u, r in owners.items() if r == rank}
        out = D.gather_recombine(local, owners, moduli, 1, rank, world, signed.shape, torch.device("cpu"))
        if rank == 0:
            q.put(bool((out[0] == signed.T).all()))
    finally:
        dist.destroy_process_group()


def test_gather_recombine_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_recombine_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert q.get(timeout=10) is True


def test_gather_units_rejects_an_unservable_plan_on_every_rank():
    plan = [[D.Unit(0, 0)], []]
    with pytest.raises(ValueError):
        D.gather_units([], plan, 1, 2)  # rank 1: no units and no template -> raises before any collective
    with pytest.raises(ValueError):
        D.gather_units([torch.zeros(2)], plan, 0, 2)  # rank 0 raises too (same plan)
