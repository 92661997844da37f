"""Multi-GPU evaluation: one process per GPU, units sharded with no
collective on the data path, one gather at the end.

The reference evaluates plaintext-CRT channels sequentially in one process
(engine.run_channels, engine.py:459-491) or as separate `hefir infer
--channel i` processes linked by files (cli.py:160-214); slot-batches are
independent evaluations.  Here a unit of work is (slot-batch, CRT channel):
units are dealt round-robin to ranks, every rank evaluates its units on its
own GPU with the unmodified single-GPU engine, and the logit ciphertexts of
all units are gathered to rank 0 (NCCL over NVLink / NVSwitch on B200s; gloo
on CPU in the tests) for decryption and CRT recombination
(engine.reconstruct_logits, engine.py:494-506).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist


@dataclass(frozen=True)
class Unit:
    batch: int    # slot-batch index
    channel: int  # plaintext-CRT channel index (index into the moduli)


def shard_plan(n_batches: int, n_channels: int, world: int) -> list:
    """Units dealt round-robin, channel-major within a batch: rank r gets
    units r, r + world, ...  Every unit appears exactly once."""
    units = [Unit(b, c) for b in range(n_batches) for c in range(n_channels)]
    return [units[r::world] for r in range(world)]


def gather_units(local: list, plan: list, rank: int, world: int, dst: int = 0, group=None):
    """Gather per-unit result tensors (all of one shape/dtype) to `dst`.

    local: tensors for plan[rank], in order.  Returns {Unit: tensor} on dst,
    None elsewhere.  Ranks with fewer units send zero padding.
    """
    if world == 1:
        return {u: t for u, t in zip(plan[0], local)}
    max_units = max(len(p) for p in plan)
    if not local:
        raise ValueError("every rank needs at least one unit (use fewer ranks)")
    shape, dtype, device = local[0].shape, local[0].dtype, local[0].device
    send = torch.zeros((max_units,) + tuple(shape), dtype=dtype, device=device)
    for i, t in enumerate(local):
        send[i].copy_(t)
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    out = {}
    for r in range(world):
        for i, u in enumerate(plan[r]):
            out[u] = bufs[r][i]
    return out


def run_units(evaluate, plan: list, rank: int, world: int, dst: int = 0, group=None):
    """Evaluate this rank's units with `evaluate(unit) -> tensor` and gather
    every unit's result to dst."""
    local = [evaluate(u) for u in plan[rank]]
    return gather_units(local, plan, rank, world, dst, group)


def recombine(results: dict, decrypt_unit, moduli, n_batches: int) -> list:
    """CRT-recombine decrypted per-channel logits into signed logits per
    batch: decrypt_unit(unit, tensor) -> (outputs, batch_size) residues mod
    moduli[unit.channel]."""
    from .engine import ChannelResult, reconstruct_logits

    moduli = tuple(int(m) for m in moduli)
    out = []
    for b in range(n_batches):
        res = None
        for c, t in enumerate(moduli):
            mat = np.asarray(decrypt_unit(Unit(b, c), results[Unit(b, c)]))
            if res is None:
                res = ChannelResult(moduli=moduli, batch_size=mat.shape[1])
            res.add(t, mat)
        out.append(reconstruct_logits(res, moduli))
    return out
