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


def _comm_device(t: torch.Tensor, group=None) -> torch.device:
    """Where a collective's buffers live: the tensor's own device, except
    CUDA tensors under gloo (which has no CUDA gather), staged through host
    memory; on B200 boxes the backend is NCCL and nothing is staged."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        return torch.device("cpu")
    return t.device


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
    cdev = _comm_device(like, group)
    send = torch.zeros((max_units,) + tuple(shape), dtype=dtype, device=cdev)
    for i, t in enumerate(local):
        send[i].copy_(t)
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    out = {}
    for r in range(world):
        for i, u in enumerate(plan[r]):
            out[u] = bufs[r][i].to(device)
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
    home = send.device
    send = send.to(_comm_device(send, group))
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == dst else None
    dist.gather(send, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    bufs = [b.to(home) for b in bufs]
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


# ---------------------------------------------------------------- CRT channels + output-channel split
#
# BASELINE config 5: CIFAR-10's 10 plaintext-CRT channels on 8 GPUs.  Dealing
# whole channels round-robin runs 2 waves (the second keeps 2 GPUs busy).
# channel_plan gives every rank floor(C / W) whole channels and splits each
# of the C mod W remaining channels over a subgroup of W // (C mod W) ranks BY
# OUTPUT CHANNEL: every rank of the subgroup computes its slice of each
# convolution's filters (then square and pool on that slice); before the next
# convolution the slices are all-gathered (NCCL over NVLink) into the full
# feature map; the dense layer on a sliced map is a partial sum over the
# rank's columns, and the partials are gathered to the subgroup root and added
# there (exact mod p; the root counts the adds like the reference's weighted
# sum).  For 10 channels on 8 GPUs every rank does 1 + 2/8 channel of work.


def channel_plan(n_channels: int, world: int):
    """-> (whole, splits): whole[r] = channels rank r evaluates alone;
    splits = [(channel, [ranks])] evaluated by output-channel slices."""
    base, rem = divmod(n_channels, world)
    whole = [[c for c in range(base * world) if c % world == r] for r in range(world)]
    splits = []
    if rem:
        size = world // rem
        for j in range(rem):
            ranks = list(range(j * size, (j + 1) * size))
            if len(ranks) == 1:
                whole[ranks[0]].append(base * world + j)
            else:
                splits.append((base * world + j, ranks))
    return whole, splits


def slices(n: int, parts: int) -> list:
    """n items in `parts` contiguous, near-equal ranges."""
    return [range(n * i // parts, n * (i + 1) // parts) for i in range(parts)]


class GpuSplitBackend:
    """Layer operations of the split program on the GPU engine."""

    def __init__(self, params, rlk):
        from . import engine as E

        self.E, self.params, self.rlk = E, params, rlk

    def conv(self, x, layer, w, counter):
        return self.E.eval_conv(x, layer, w, self.params, counter)

    def square(self, x, counter):
        return self.E.eval_square(x, self.rlk, self.params, counter)

    def pool(self, x, layer, counter):
        return self.E.eval_pool(x, layer, self.params, counter)

    def fc(self, x, layer, w, counter):
        return self.E.eval_fc(x, layer, w, self.params, counter)

    def wrap(self, shape, data, delta):
        return self.E.GpuCipherTensor(shape, data, delta, self.params.t, self.params)

    def add(self, a, b):
        from . import ops

        return ops.hadd_device(self.E.context_for(self.params, a.device), a, b)


def _split_program(x, model, backend, S: int, me: int, counter):
    """One CRT channel's network, rank `me` of an S-rank subgroup (a
    generator: it yields ("all_gather", tensor) / ("gather", tensor) at the
    collectives and receives the list of every rank's tensor, or None on
    non-root ranks for "gather").  Returns the logits on rank 0 of the
    subgroup, None elsewhere."""
    from dataclasses import replace

    from .nn import kind_of

    layers = list(zip(model.spec.layers, model.weights))
    if not layers or kind_of(layers[0][0]) != "conv":
        raise ValueError("the output-channel split starts at a convolution")
    cut = None  # channel slices of every rank while x holds only this rank's slice

    def join(x):
        h, w, c = x.shape
        cmax = max(len(s) for s in cut)
        d = x.data.reshape((h * w, c) + tuple(x.data.shape[1:]))
        if c < cmax:
            d = torch.cat([d, d.new_zeros((h * w, cmax - c) + tuple(d.shape[2:]))], dim=1)
        chunks = yield ("all_gather", d.contiguous())
        full = torch.cat([ch[:, :len(s)] for ch, s in zip(chunks, cut)], dim=1)
        C = sum(len(s) for s in cut)
        return backend.wrap((h, w, C), full.reshape((h * w * C,) + tuple(d.shape[2:])).contiguous(), x.delta)

    for layer, wts in layers:
        k = kind_of(layer)
        if k == "conv":
            if layer.groups != 1:
                raise ValueError("the output-channel split needs dense convolutions")
            if cut is not None:
                x = yield from join(x)
            cut = slices(layer.filters, S)
            mine = cut[me]
            x = backend.conv(x, replace(layer, filters=len(mine)), np.asarray(wts)[mine.start:mine.stop], counter)
        elif k == "square":
            x = backend.square(x, counter)
        elif k == "pool":
            x = backend.pool(x, layer, counter)
        elif k == "fc" and cut is not None:
            h, w, _ = x.shape
            C = sum(len(s) for s in cut)
            W = np.asarray(wts)
            cols = [np.array([(y * w + xx) * C + ch for y in range(h) for xx in range(w) for ch in s], dtype=np.int64)
                    for s in cut]
            part = backend.fc(x, layer, W[:, cols[me]], counter)
            parts = yield ("gather", part.data)
            if me != 0:
                return None
            acc = parts[0]
            for p in parts[1:]:
                acc = backend.add(acc, p)
            # the adds of the partials, counted as the reference counts a weighted
            # sum's adds (engine.py:206-223): one per extra non-empty partial
            nz = np.stack([(W[:, c] != 0).any(axis=1) for c in cols]).sum(axis=0)
            counter.hadd += int(np.maximum(nz - 1, 0).sum())
            x = backend.wrap((1, 1, W.shape[0]), acc, part.delta)
            cut = None
        elif k == "fc":
            if me != 0:
                return None
            x = backend.fc(x, layer, wts, counter)
    if cut is not None:
        x = yield from join(x)
        if me != 0:
            return None
    return x


def run_split_emulated(x, model, backend, S: int, counters=None):
    """Run all S ranks of a split program in lockstep in ONE process (one
    GPU): the collectives are resolved in memory.  Returns rank 0's logits."""
    counters = counters if counters is not None else [None] * S
    from .engine import OpCounter

    counters = [c if c is not None else OpCounter() for c in counters]
    gens = [_split_program(x, model, backend, S, r, counters[r]) for r in range(S)]
    msgs = [None] * S
    results = [None] * S
    alive = list(range(S))
    while alive:
        ops_ = {}
        for r in alive:
            try:
                ops_[r] = gens[r].send(msgs[r])
            except StopIteration as stop:
                results[r] = stop.value
        alive = [r for r in alive if r in ops_]
        if not alive:
            break
        kinds = {ops_[r][0] for r in alive}
        if len(kinds) != 1 or len(alive) != S:
            raise RuntimeError("split ranks diverged")
        data = [ops_[r][1] for r in range(S)]
        kind = kinds.pop()
        for r in range(S):
            msgs[r] = list(data) if kind == "all_gather" or r == 0 else None
    return results[0]


def run_split(x, model, backend, ranks: list, rank: int, group=None, counter=None):
    """Run this rank's part of a split program with torch.distributed
    collectives over `group` (the subgroup of `ranks`).  Returns the logits
    on ranks[0], None elsewhere."""
    S, me = len(ranks), ranks.index(rank)
    gen = _split_program(x, model, backend, S, me, counter)
    msg = None
    while True:
        try:
            kind, data = gen.send(msg)
        except StopIteration as stop:
            return stop.value
        home = data.device
        data = data.to(_comm_device(data, group))
        if kind == "all_gather":
            lst = [torch.empty_like(data) for _ in range(S)]
            dist.all_gather(lst, data, group=group)
        else:
            lst = [torch.empty_like(data) for _ in range(S)] if me == 0 else None
            dist.gather(data, lst, dst=ranks[0], group=group)
        msg = [t.to(home) for t in lst] if lst is not None else None


def split_groups(splits):
    """torch.distributed subgroups of a channel_plan's splits (every rank must
    call this, in the same order)."""
    return [dist.new_group(ranks) for _, ranks in splits]


# ---------------------------------------------------------------- decrypt, gather, recombine


def decrypt_residues(logits, sk, params, batch_size: int) -> torch.Tensor:
    """Decrypt + slot-decode a logits GpuCipherTensor on its own GPU:
    DEVICE int64 (outputs, batch) residues mod t (engine.py:178-192)."""
    from . import engine as E

    polys = E.decrypt_device(logits, sk, params)
    slots = E.codec_for(params.t, params.ring_degree, logits.data.device).decode(polys)
    return slots[:, :batch_size].contiguous()


def gather_recombine(local: dict, owners: dict, moduli, n_batches: int, rank: int, world: int, shape, device,
                     dst: int = 0, group=None, lazy: bool = False):
    """The pipeline's one exchange: every rank holds the decrypted residues
    (DEVICE int64 (outputs, batch)) of the (batch, channel) units it owns
    (`local`: {Unit: tensor}); `owners` maps every Unit to its rank (identical
    on all ranks).  The residue matrices are gathered to dst (NCCL; 8 x 10 x
    8192 x 8 B per CIFAR batch instead of the 66 MB of logit ciphertexts) and
    CRT-recombined there on the GPU.  `shape` = (outputs, batch) of one
    matrix and `device` this rank's device (ranks that own no unit still take
    part in the gather).  Returns the signed logits [(batch, outputs) object
    array per slot-batch] on dst, None elsewhere; lazy=True returns the
    engine.DeviceCrtValues instead (no host synchronisation; .values().T is
    the (batch, outputs) array)."""
    from .engine import ChannelResult, reconstruct_logits, reconstruct_logits_device

    units = sorted(owners, key=lambda u: (u.batch, u.channel))
    plan = [[u for u in units if owners[u] == r] for r in range(world)]
    mine = [local[u] for u in plan[rank]]
    template = torch.empty(tuple(shape), dtype=torch.int64, device=device)
    res = gather_units(mine, plan, rank, world, dst, group, template=template)
    if rank != dst:
        return None
    moduli = tuple(int(m) for m in moduli)
    out = []
    for b in range(n_batches):
        if lazy and res[Unit(b, 0)].is_cuda:
            out.append(reconstruct_logits_device([res[Unit(b, c)] for c in range(len(moduli))], moduli))
            continue
        cr = ChannelResult(moduli=moduli, batch_size=int(res[Unit(b, 0)].shape[1]))
        for c, t in enumerate(moduli):
            cr.add(t, res[Unit(b, c)])
        out.append(reconstruct_logits(cr, moduli))
    return out
