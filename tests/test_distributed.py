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
