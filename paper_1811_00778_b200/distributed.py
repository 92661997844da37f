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


def gather_units(local: list, plan: list, rank: int, world: int, dst: int = 0, group=None,
                 template: torch.Tensor | None = None):
    """Gather per-unit result tensors (all of one shape/dtype) to `dst`.

    local: tensors for plan[rank], in order.  Returns {Unit: tensor} on dst,
    None elsewhere.  Ranks with fewer units send zero padding; a rank with
    no units needs `template` (a tensor of the unit shape/dtype/device).
    The plan is identical on every rank, so a plan this call cannot serve is
    rejected on every rank before any collective starts (no rank is left
    waiting inside the gather).
    """
    if len(plan) != world:
        raise ValueError(f"plan has {len(plan)} ranks, world is {world}")
    if len(local) != len(plan[rank]):
        raise ValueError(f"rank {rank}: {len(local)} results for {len(plan[rank])} units")
    if world == 1:
        return {u: t for u, t in zip(plan[0], local)}
    max_units = max(len(p) for p in plan)
    if min(len(p) for p in plan) == 0 and template is None:
        raise ValueError("a rank of the plan has no units: pass `template` (or use fewer ranks)")
    like = local[0] if local else template
    shape, dtype, device = like.shape, like.dtype, like.device
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


# ---------------------------------------------------------------- output-channel groups
#
# SURVEY §8(e) partitioning (3): in the MNIST HCNN the second convolution is
# grouped (nn_oracle.py:122, groups = the first convolution's filter count), so
# conv1 filter g -> square -> conv2 group g -> square is independent of every
# other g until the dense layer.  Each rank evaluates its groups on the whole
# (replicated) input; the dense layer, being linear, splits into per-rank
# partial sums over the rank's channels, and one gather + modular adds on
# rank 0 finish it.  This shards ONE slot-batch (strong scaling).


def groupable(spec) -> int:
    """Number of independent output-channel groups of a conv-square-grouped
    conv-square-fc network, or 0 if the network does not have that shape."""
    from .nn import kind_of

    kinds = [kind_of(layer) for layer in spec.layers]
    if kinds != ["conv", "square", "conv", "square", "fc"]:
        return 0
    c1, c2 = spec.layers[0], spec.layers[2]
    if c1.groups != 1 or c2.groups != c1.filters or spec.input_shape[2] != 1:
        return 0
    return c1.filters


def group_plan(groups: int, world: int) -> list:
    """Groups dealt round-robin to ranks (ranks beyond `groups` get none)."""
    return [list(range(r, groups, world)) for r in range(world)]


def slice_model(model, sel: list):
    """Sub-network of the groups in `sel` (sorted): conv1 filters sel, conv2
    filters of those groups (groups = len(sel)), dense-layer columns of their
    channels.  Its logits are this rank's partial sums of the full logits."""
    from .nn import NetworkSpec, QuantizedModel, layer_shapes

    spec = model.spec
    G = groupable(spec)
    if not G or not sel:
        raise ValueError("network is not group-shardable or the selection is empty")
    c1, sq1, c2, sq2, fc = spec.layers
    per = c2.filters // c2.groups
    w1, _, w2, _, wf = model.weights
    w1s = np.asarray(w1)[sel]
    chans = [g * per + k for g in sel for k in range(per)]
    w2s = np.asarray(w2)[chans]
    h, w, c = layer_shapes(spec)[3]  # after square2: (h, w, c2.filters)
    wf = np.asarray(wf, dtype=object if np.asarray(wf).dtype == object else np.int64)
    cols = [(y * w + x) * c + ch for y in range(h) for x in range(w) for ch in chans]
    wfs = wf[:, cols]
    from dataclasses import replace

    layers = (replace(c1, filters=len(sel)), sq1, replace(c2, filters=len(chans), groups=len(sel)), sq2, fc)
    sub = NetworkSpec(spec.name + f"[groups {sel}]", spec.input_shape, spec.input_scale, layers, spec.wide_values)
    return QuantizedModel(spec=sub, bit_width=model.bit_width, weights=[w1s, None, w2s, None, wfs])


def eval_network_groups(tensor, model, rlk, params, rank: int, world: int, counter=None, dst: int = 0,
                        group=None):
    """engine.eval_network of one slot-batch sharded by output-channel group.

    Every rank holds the whole input; rank r evaluates the groups of
    group_plan(G, world)[r] and produces partial logits; the partials are
    gathered to dst (NCCL) and added there with the library's modular add
    (hadd, counted like the reference counts the adds of a weighted sum, so
    the OpCounters of all ranks sum to the single-GPU counter).  Returns the
    logits GpuCipherTensor on dst, None elsewhere."""
    from . import engine as E

    counter = counter if counter is not None else E.OpCounter()
    G = groupable(model.spec)
    if not G:
        raise ValueError("network is not group-shardable")
    plan = group_plan(G, world)
    active = [r for r in range(world) if plan[r]]
    sel = plan[rank]
    part = None
    if sel:
        part = E.eval_network(tensor, slice_model(model, sel), rlk, params, counter)
    if world == 1:
        return part
    n_out = model.spec.layers[-1].filters
    g = E.context_for(params, tensor.data.device)
    send = part.data if part is not None else g.empty(n_out)
    if part is None:
        send.zero_()
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    from . import ops

    acc = bufs[active[0]]
    for r in active[1:]:
        acc = ops.hadd_device(g, acc, bufs[r])
    if counter is not None:
        counter.hadd += n_out * (len(active) - 1)
    return E.GpuCipherTensor((1, 1, n_out), acc, output_delta(model.spec, tensor.delta), params.t, params)


def output_delta(spec, delta: int) -> int:
    """Scale of the logits: conv / fc multiply by the weight scale, square
    squares, pool multiplies by the window size (engine.py:237-397)."""
    from .nn import kind_of

    for layer in spec.layers:
        k = kind_of(layer)
        if k in ("conv", "fc"):
            delta *= layer.weight_scale
        elif k == "square":
            delta = delta * delta
        elif k == "pool":
            delta *= layer.extent * layer.extent
    return delta
