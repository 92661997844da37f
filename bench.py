#!/usr/bin/env python3
"""HCNN encrypted-batch benchmark on B200 (BASELINE.json metric).

Workload (default): the MNIST HCNN (conv-square-conv-square-fc, nn_oracle.py:
108-126) at the paper's >80-bit parameter set 1 (N = 2^13, 11 x 30-bit primes,
log q = 330, t = 5522259017729, presets.py:62-69), ONE full slot-batch of 8192
synthetic 28x28 images (scale-4 pixels), dense random 4-bit weights (every tap
executes).  One step = one homomorphic evaluation of the whole network over
the batch (engine.eval_network), 1520 HSquares + 46,000 plaintext MACs.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one process per GPU): every rank evaluates its own
independent slot-batch (weak scaling); the logit ciphertexts are gathered to
rank 0 with NCCL at the end of each step (the final-gather step of the
pipeline).  `value` = images of all ranks / max-over-ranks step time.

`--impl reference` times the reference algorithm on the host CPU (the pinned
oracle port in oracle/, all host cores) on a bounded sample and extrapolates
to the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "HCNN encrypted-batch latency (s) and images/s, MNIST/CIFAR-10, at 1/2/4/8 B200"
SET1_PRIMES = (1073643521, 1073479681, 1073184769, 1073053697, 1072857089, 1072496641,
               1071513601, 1071415297, 1071087617, 1070727169, 1070432257)
MNIST_T = 5522259017729


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--seed", type=int, default=2024)
    ap.add_argument("--profile-only", action="store_true", help="one step, no timing (for ncu)")
    ap.add_argument("--workload", default="mnist", choices=["mnist", "mnist3", "cifar"])
    ap.add_argument("--channels", type=int, default=None,
                    help="use only the first K plaintext-CRT channels (tests; the metric uses all)")
    ap.add_argument("--shard", default="units", choices=["units", "groups"],
                    help="units: one slot-batch (x CRT channel) per rank, weak scaling; groups: one MNIST "
                         "slot-batch split over the ranks by output-channel group, strong scaling")
    return ap.parse_args()


# ---------------------------------------------------------------- workload


WORKLOADS = {
    "mnist": dict(preset="1", net="mnist_hcnn", image=(28, 28, 1), pix=5, delta=4,
                  desc="MNIST HCNN, preset 1 (N=8192, 11x30-bit primes, log q 330, t=5522259017729), "
                       "one 8192-image slot-batch per GPU"),
    "mnist3": dict(preset="3", net="mnist_hcnn", image=(28, 28, 1), pix=5, delta=4,
                   desc="MNIST HCNN, preset 3 (N=16384, 11 primes, t=5522259017729), one 16384-image slot-batch per GPU"),
    "cifar": dict(preset="5", net="cifar10_hcnn", image=(32, 32, 3), pix=256, delta=255,
                  desc="CIFAR-10 HCNN, preset 5 (N=8192, 10 primes, log q 300, 10 plaintext-CRT channels "
                       "t_i ~ 2^22), one 8192-image batch; the 10 channels are dealt round-robin over the GPUs"),
}


def build_workload(name: str, rank: int, world: int, seed: int, channels: int | None = None):
    """This rank's units of one step: (params, rlk, model, device input) per
    (slot-batch, CRT channel).  MNIST: one batch per rank (replicas);
    CIFAR: the 10 channels of one batch, distributed.channel_plan: whole
    channels per rank plus the leftover channels split by output channel
    over subgroups (10 on 8 GPUs: 1 whole + 1/4 of a split channel each)."""
    from paper_1811_00778_b200 import bfv as B
    from paper_1811_00778_b200 import distributed as D
    from paper_1811_00778_b200 import engine as E
    from paper_1811_00778_b200 import nn, presets

    w = WORKLOADS[name]
    preset = presets.load_preset(w["preset"])
    n = preset.ring_degree
    spec = nn.NETWORKS[w["net"]]()
    model = nn.random_model(spec, np.random.default_rng(seed + 1))
    splits = []
    n_ch = min(preset.channels, channels or preset.channels)
    if n_ch == 1 and preset.channels == 1:
        whole = [[D.Unit(r, 0)] for r in range(world)]
        n_batches = world
    else:
        wc, sp = D.channel_plan(n_ch, world)
        whole = [[D.Unit(0, c) for c in wc[r]] for r in range(world)]
        splits = [(D.Unit(0, c), ranks) for c, ranks in sp]
        n_batches = 1
    owners = {u: r for r in range(world) for u in whole[r]}
    owners.update({u: ranks[0] for u, ranks in splits})
    mine = list(whole[rank]) + [u for u, ranks in splits if rank in ranks]
    units = []
    t0 = time.time()
    for u in mine:
        params = presets.build_context(preset, u.channel)
        sk, pk, rlk = B.keygen(params, np.random.default_rng(seed + 10 * u.channel))
        irng = np.random.default_rng(seed + 100 + u.batch)
        images = list(irng.integers(0, w["pix"], (n,) + w["image"]))
        enc = B.SlotEncoder(params.t, n)
        gin = E.pack_images_device(images, E.PackingLayout(n, n), enc, pk, params,
                                   np.random.default_rng(seed + 200 + 31 * u.batch + u.channel),
                                   delta=w["delta"])
        split = next((ranks for v, ranks in splits if v == u), None)
        units.append(dict(unit=u, params=params, sk=sk, rlk=rlk, gin=gin, enc=enc, split=split,
                          model=E.reduce_model(model, params.t), images=images))
    return dict(units=units, owners=owners, splits=splits, n_batches=n_batches, images_per_step=n * n_batches,
                moduli=tuple(int(t) for t in preset.plaintext_moduli[:n_ch]),
                setup_s=time.time() - t0, desc=w["desc"], spec=spec, preset=preset)


# ---------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi style sampling through NVML during the timed region."""

    def __init__(self, index: int):
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except Exception:
                    r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.th.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------- work model


def ntt_butterflies(name: str, K: int, KP: int, D: int, N: int, cts: float):
    """NTT butterflies of one launch of an NTT kernel over `cts` ciphertexts."""
    bfly = (N // 2) * (N.bit_length() - 1)
    if name == "k_tensor":
        return (K + KP) * 5 * bfly * cts
    if name == "k_relin":
        return K * (D + 2) * bfly * cts
    if name == "k_rb_fwd":  # D digit transforms mod each of the 3 primes of R
        return 3 * D * bfly * cts
    if name == "k_rb_inv":  # 2 parts x 3 primes of R inverse transforms per q_j
        return 6 * K * bfly * cts
    return None


def s8d_modmuls(name: str, K: int, KP: int, D: int, N: int, cts: float, logq: int = 330):
    """SURVEY.md section 8(d)'s work formula, in modular-multiply equivalents
    (1 per NTT butterfly, per pointwise product, per base-conversion term),
    split over the kernels that do the work; 3 IMAD per modmul (Shoup)."""
    B = (N // 2) * (N.bit_length() - 1)
    L = K + KP
    name = name[:-3] if name.endswith("_tc") else name  # same work, tensor-core dots
    if name == "k_tensor":  # 2 fwd + 3 inv NTTs over Q u P, 3 pointwise products
        m = (2 * L + 3 * L) * B + 3 * L * N
    elif name == "k_relin":  # D fwd + 2 inv NTTs over Q, 2 D pointwise MACs
        m = (D * K + 2 * K) * B + 2 * D * K * N
    elif name == "k_extend":  # Q -> P of 2 parts
        m = 2 * K * KP * N
    elif name == "k_scale":  # 3 parts Q -> P -> Q, digits of c2
        m = 6 * K * KP * N + K * ((logq + 31) // 32) * N
    else:
        return None
    return m * cts


def kernel_work(name: str, K: int, KP: int, D: int, N: int, cts: float):
    """Algorithmic (HBM bytes, IMAD issue slots) of one launch over `cts`
    ciphertexts.

    IMAD slots: the integer multiplier (fmaheavy pipe) issues a 32-bit IMAD in
    one slot and IMAD.HI / IMAD.WIDE in two (measured: 18.4 vs 9.0 T/s), so a
    Shoup butterfly costs 4 slots, a lazy 64-bit multiply-accumulate 2, a
    Shoup modmul 4, a Barrett-64 modmul 8, a Montgomery REDC 3.  Bytes are
    the compulsory DRAM reads + writes of the kernel's operands (u32
    residues); keys and twiddles are L2-resident and counted once per launch.
    """
    logn = N.bit_length() - 1
    bfly = (N // 2) * logn
    L = K + KP
    if name == "k_scale_tc":  # the dot products on the tensor cores; per part: K Shoup + fixed
        # point, KP x (REDC + 2 Shoup + fixed point), K x REDC on the integer pipe
        part = K * 4 + K * 2 + KP * (3 + 2 * 4 + 2) + K * 3
        digits = K * 4 + K * 2 + (K + 1) * (K * 2 + 2)
        return 4 * N * (3 * L + 3 * K + D) * cts, N * (3 * part + digits) * cts
    if name == "k_extend_tc":  # per part: K Shoup, fixed point, KP x REDC (dots on the tensor cores)
        return 4 * N * 2 * (K + KP) * cts, 2 * N * (K * 4 + K * 2 + KP * 3) * cts
    if name == "k_tensor":  # 2 fwd + 3 inv NTT per prime, 3 products, N^-1 scaling
        slots = L * (5 * bfly * 4 + 3 * N * 8 + 3 * N * 4)
        byts = L * N * 4 * (2 + 3)
        fixed = L * N * 16
    elif name == "k_relin":  # D fwd + 2 inv NTT per prime, 2D lazy MACs, N^-1
        slots = K * ((D + 2) * bfly * 4 + 2 * D * N * 2 + 2 * N * 4)
        byts = 4 * N * (D + 2 * K + 2 * K)
        fixed = 4 * N * 2 * D * K + K * N * 16
    elif name == "k_scale":  # per part: K Shoup, Q->P (K MAC + REDC) x KP, 3 Shoup x KP, P->Q
        part = K * 4 + KP * (K * 2 + 3 * 2) + KP * 4 * 2 + K * (KP * 2 + 3 * 2) + (K + KP) * 2
        digits = K * 4 + K * 2 + (K + 1) * (K * 2 + 2)
        slots = N * (3 * part + digits)
        byts = 4 * N * (3 * L + 3 * K + D)
        fixed = 0
    elif name == "k_extend":  # per part: K Shoup, fixed point, KP x (K MAC + REDC)
        slots = 2 * N * (K * 4 + K * 2 + KP * (K * 2 + 3))
        byts = 4 * N * 2 * (K + KP)
        fixed = 0
    elif name == "k_rb_fwd":  # relinearisation over R: D forward NTTs mod 3 primes
        slots = 3 * D * bfly * 4
        byts = 4 * N * (D + 3 * D)
        fixed = 0
    elif name == "k_rb_mac_tc":  # the products on the tensor cores; a REDC per output on the integer pipe
        slots = 3 * 2 * K * N * 4
        byts = 4 * N * (3 * D + 6 * K)
        fixed = 3 * N * 96 * 96
    elif name == "k_rb_mac":  # 3 x 2K x D lazy 64-bit MACs per coefficient, a fold per output
        slots = 3 * 2 * K * N * (D * 2 + 7)
        byts = 4 * N * (3 * D + 6 * K)
        fixed = 4 * N * 3 * D * 2 * K
    elif name == "k_rb_inv":  # 6 inverse NTTs per q_j, CRT (4 MACs + REDC) per output
        slots = K * (6 * bfly * 4 + 2 * N * 12)
        byts = 4 * N * (6 * K + 2 * K + 2 * K)
        fixed = 0
    else:
        return None
    return byts * cts + fixed, slots * cts


# ---------------------------------------------------------------- our arm


def g0_bytes(units) -> int:
    """bytes of one u32 ciphertext part of the workload (K x N x 4)"""
    d = units[0]["gin"].data
    return int(d.shape[2] * d.shape[3] * 4)


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1811_00778_b200 import _lib
    from paper_1811_00778_b200 import distributed as D
    from paper_1811_00778_b200 import engine as E

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())  # (oversubscribed tests)
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("HCNN_DIST_BACKEND", "nccl")  # gloo: multi-rank logic on one GPU (tests)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    groups = args.shard == "groups"
    if groups and args.workload not in ("mnist", "mnist3"):
        raise SystemExit("--shard groups needs a grouped network (mnist, mnist3)")
    # groups: every rank holds the same slot-batch and evaluates its share of it
    W = build_workload(args.workload, 0 if groups else rank, 1 if groups else world, args.seed, args.channels)
    units = W["units"]
    ctxs = [E.context_for(u["params"]) for u in units]
    counters = []
    split_pgs = D.split_groups([(u.channel, ranks) for u, ranks in W["splits"]]) if world > 1 and not groups else []
    split_pg = {u: pg for (u, _), pg in zip(W["splits"], split_pgs)}
    n_img = W["preset"].ring_degree
    n_out = W["spec"].layers[-1].filters
    dev = torch.device("cuda", local)

    def evaluate(u, x=None):
        counter = E.OpCounter()
        x = x if x is not None else u["gin"]
        if groups:
            out = D.eval_network_groups(x, u["model"], u["rlk"], u["params"], rank, world, counter)
        elif u["split"] is not None:
            out = D.run_split(x, u["model"], D.GpuSplitBackend(u["params"], u["rlk"]), u["split"], rank,
                              split_pg.get(u["unit"]), counter)
        else:
            out = E.eval_network(x, u["model"], u["rlk"], u["params"], counter)
        counters.append(counter)
        return out

    def finish(outs):
        """The pipeline's last step: decrypt each logits tensor on the GPU that
        owns it, gather the plaintext residues to rank 0 (NCCL), CRT-recombine
        there on the GPU."""
        local = {}
        for u, o in zip(units, outs):
            if o is not None:
                local[u["unit"]] = D.decrypt_residues(o, u["sk"], u["params"], n_img)
        if groups:
            if rank != 0:
                return None
            owners = {D.Unit(0, 0): 0}
            return D.gather_recombine(local, owners, W["moduli"], 1, 0, 1, (n_out, n_img), dev, lazy=True)
        return D.gather_recombine(local, W["owners"], W["moduli"], W["n_batches"], rank, world, (n_out, n_img), dev,
                                  lazy=True)

    def step(inputs=None):
        counters.clear()
        outs = [evaluate(u, None if inputs is None else inputs[i]) for i, u in enumerate(units)]
        return finish(outs)

    if args.profile_only:
        step()
        torch.cuda.synchronize()
        return

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device-resident inputs, larger than L2 each step)
    stream = torch.cuda.current_stream()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    L = _lib.lib()
    for g in ctxs:
        _lib.check(L.hcnn_profile(g.handle, 1))
    launches0 = sum(g.launches() for g in ctxs)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        h0 = time.perf_counter()
        for _ in range(args.steps):
            outs = step()
        host_issue_ms = (time.perf_counter() - h0) * 1e3 / args.steps  # host time to enqueue a step
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = sum(g.launches() for g in ctxs) - launches0
    step_counters = list(counters[-len(units):])  # the last timed step's counters (one per unit)
    # the last step's signed logits, read on the host after the timed region
    result_shape = list(outs[0].values().T.shape) if (rank == 0 and outs) else None
    ms = ev0.elapsed_time(ev1) / args.steps
    prof = {}
    for g in ctxs:
        for name, (cnt, tot) in g.profile_read().items():
            c0, t0 = prof.get(name, (0, 0.0))
            prof[name] = (c0 + cnt, t0 + tot)
        _lib.check(L.hcnn_profile(g.handle, 0))
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- end to end through the public API: pinned host u32 ciphertexts in,
    # logits out, copies inside the timed region
    host_in = []
    for u in units:
        h = torch.empty(u["gin"].data.shape, dtype=torch.int32, pin_memory=True)
        h.copy_(u["gin"].data)
        host_in.append(h)
    e2e_steps = max(3, args.steps)
    n_out = W["spec"].layers[-1].filters
    host_out = [[torch.empty((n_out,) + tuple(u["gin"].data.shape[1:]), dtype=torch.int32, pin_memory=True)
                 for _ in range(e2e_steps)] for u in units]
    def e2e_run(k):
        for u, h, ho in zip(units, host_in, host_out):
            if groups or u["split"] is not None:  # upload, sharded evaluation, logits back on the root
                for i in range(k):
                    x = E.GpuCipherTensor(u["gin"].shape, h.to("cuda", non_blocking=True), u["gin"].delta,
                                          u["gin"].channel_modulus, u["params"])
                    o = evaluate(u, x)
                    if o is not None:
                        ho[i % len(ho)].copy_(o.data, non_blocking=True)
            else:  # public serving API: uploads of step s+1 overlap the evaluation of step s
                E.eval_network_stream([h] * k, u["model"], u["rlk"], u["params"], u["gin"].shape,
                                      u["gin"].delta, E.OpCounter(), outputs=ho)

    e2e_run(max(args.warmup, 2))  # warm-up: streams, input buffers, pinned pages
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    w0 = time.perf_counter()
    e0.record(stream)
    e2e_run(e2e_steps)
    e1.record(stream)
    torch.cuda.synchronize()
    wall_e2e = (time.perf_counter() - w0) / e2e_steps
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # ---- end to end through the reference-facing drop-in: the reference's
    # host objects (CipherTensor of Ciphertexts of int64 RingElems) in,
    # host CipherTensor out, one engine.eval_network call per step
    dropin = None
    if not groups and args.workload != "cifar":  # (CIFAR's host objects would be ~40 GB of int64)
        host_cts = [u["gin"].to_host() for u in units]  # untimed: the caller's objects
        def dropin_run(k):
            for _ in range(k):
                for u, hc in zip(units, host_cts):
                    o = E.eval_network(hc, u["model"], u["rlk"], u["params"], E.OpCounter())
            return o

        dropin_run(2)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        d0 = torch.cuda.Event(enable_timing=True)
        d1 = torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        d0.record(stream)
        last = dropin_run(e2e_steps)
        d1.record(stream)
        torch.cuda.synchronize()
        wall_d = (time.perf_counter() - w0) / e2e_steps
        d_ms = d0.elapsed_time(d1) / e2e_steps
        if world > 1:
            t = torch.tensor([d_ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            d_ms = float(t.item())
        in64 = sum(len(hc.cts) * 2 * hc.cts[0].parts[0].residues.nbytes for hc in host_cts)
        dropin = {"value": round(W["images_per_step"] / (d_ms / 1e3), 2), "unit": "images/s",
                  "ms_per_step": round(d_ms, 3), "wall_ms_per_step": round(wall_d * 1e3, 3),
                  "h2d_bytes_per_step": int(sum(u["gin"].data.numel() * 4 for u in units)),
                  "host_bytes_read_per_step": int(in64),
                  "d2h_bytes_per_step": int(len(last.cts) * 2 * g0_bytes(units)),
                  "path": "engine.eval_network(host CipherTensor of int64 RingElems) -> host CipherTensor: "
                          "residues narrowed to u32 by a thread pool into a reused pinned buffer, by row bands, "
                          "each band uploaded and the conv1/square1/conv2/square2 wavefront advanced on it while the next band is narrowed",
                  "steps": e2e_steps}
        del host_cts

    if rank != 0:
        dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "MEASURED_PEAKS.json" if "hbm_gbs" in peaks else "fallback"
    import ctypes

    imad = ctypes.c_double()
    _lib.check(L.hcnn_int_peak(local, 0, ctypes.byref(imad)))
    imad_peak = imad.value / 1e12
    total_ms = sum(v[1] for v in prof.values())
    dom = max(prof, key=lambda k: prof[k][1]) if prof else None
    roof = None
    kernels = {name: {"launches": cnt, "ms_total": round(tot, 4), "share": round(tot / total_ms, 4)}
               for name, (cnt, tot) in prof.items()}
    n_sq = sum(c.hsquare for c in step_counters) * args.steps
    g0 = ctxs[0]
    if dom:
        cnt, tot = prof[dom]
        work = kernel_work(dom, g0.K, g0.KP, g0.D, g0.N, n_sq / cnt)
        avg_s = tot / cnt / 1e3
        if work:
            byts, ops = work
            gbs = byts / avg_s / 1e9
            tops = ops / avg_s / 1e12
            hbm_frac = gbs / hbm_peak
            int_frac = tops / imad_peak
            traffic = None
            try:
                with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
                    per_ct = json.load(fh).get(dom)
                traffic = round(per_ct * (n_sq / cnt)) if per_ct and args.workload == "mnist" else None
            except Exception:
                pass
            int_bound = int_frac >= hbm_frac
            roof = {
                "kernel": dom,
                "bound": "int" if int_bound else "hbm",
                "achieved": round(tops if int_bound else gbs, 3),
                "peak": round(imad_peak if int_bound else hbm_peak, 3),
                "unit": "T IMAD-slots/s" if int_bound else "GB/s",
                "frac": round(int_frac if int_bound else hbm_frac, 4),
                "traffic": traffic,
                "hbm": {"achieved_gbs": round(gbs, 1), "peak_gbs": hbm_peak, "frac": round(hbm_frac, 4),
                        "peak_source": hbm_src + " (of measured)", "algorithmic_bytes_per_launch": byts},
                "int": {"achieved_t_slots_s": round(tops, 3), "peak_t_slots_s": round(imad_peak, 3),
                        "frac": round(int_frac, 4),
                        "peak_source": "measured in bench.py (hcnn_int_peak: 32-bit IMAD issue rate, fmaheavy pipe)",
                        "imad_slots_per_launch": ops},
                "avg_launch_ms": round(avg_s * 1e3, 4),
                "share_of_step": round(tot / total_ms, 4),
                "note": "integer-pipe kernel (NTT butterflies); the base conversions around it run on the tensor cores (k_extend_tc, k_scale_tc: DESIGN.md section 4.2)",
            }
            mm = s8d_modmuls(dom, g0.K, g0.KP, g0.D, g0.N, n_sq / cnt)
            if mm:
                ach = 3 * mm / avg_s / 1e12
                roof["s8d"] = {
                    "modmul_per_launch": mm, "achieved_t_imad_s": round(ach, 3),
                    "peak_t_imad_s": round(imad_peak, 3), "frac": round(ach / imad_peak, 4),
                    "note": "SURVEY.md 8(d) work formula: modmul-equivalents x 3 IMAD over the measured 32-bit IMAD rate",
                }
            nb = ntt_butterflies(dom, g0.K, g0.KP, g0.D, g0.N, n_sq / cnt)
            if nb:
                bf = ctypes.c_double()
                _lib.check(L.hcnn_int_peak(local, 8, ctypes.byref(bf)))
                ach = nb / avg_s / 1e12
                roof["bfly"] = {
                    "achieved_t_bfly_s": round(ach, 3), "peak_t_bfly_s": round(bf.value / 1e12, 3),
                    "frac": round(ach / (bf.value / 1e12), 4), "butterflies_per_launch": nb,
                    "peak_source": "measured in bench.py (hcnn_int_peak kind 8: register-resident Harvey "
                                   "butterflies, the NTT's instruction mix; attainable peak of the integer pipes)",
                    "note": "counts NTT butterflies only (the kernel's MACs and exchanges are extra work)",
                }

    # every kernel's fraction of its roofline (HBM bytes and 8(d) IMAD work)
    for name, (cnt, tot) in prof.items():
        avg_s = tot / cnt / 1e3
        wk = kernel_work(name, g0.K, g0.KP, g0.D, g0.N, n_sq / cnt)
        mm = s8d_modmuls(name, g0.K, g0.KP, g0.D, g0.N, n_sq / cnt)
        if wk:
            kernels[name]["hbm_frac"] = round(wk[0] / avg_s / 1e9 / hbm_peak, 4)
            kernels[name]["imad_slot_frac"] = round(wk[1] / avg_s / 1e12 / imad_peak, 4)
        if mm:
            kernels[name]["s8d_frac"] = round(3 * mm / avg_s / 1e12 / imad_peak, 4)
    # the relinearisation over R as one stage (its three kernels) against the
    # 8(d) relinearisation work of the reference algorithm
    rb = [n for n in ("k_rb_fwd", "k_rb_mac", "k_rb_mac_tc", "k_rb_inv") if n in prof]
    if len(rb) == 3:
        cnt = prof["k_rb_fwd"][0]
        tot = sum(prof[n][1] for n in rb)
        mm = s8d_modmuls("k_relin", g0.K, g0.KP, g0.D, g0.N, n_sq / cnt)
        avg_s = tot / cnt / 1e3
        kernels["relin_rbasis"] = {"kernels": rb, "launches": cnt, "ms_total": round(tot, 4),
                                   "share": round(tot / total_ms, 4),
                                   "s8d_frac": round(3 * mm / avg_s / 1e12 / imad_peak, 4),
                                   "note": "8(d) relinearisation work (D K + 2K NTTs, 2 D K N MACs) over the "
                                           "three kernels' time"}
    images = W["images_per_step"]
    value = images / (ms / 1e3)
    in_bytes = int(sum(h.numel() for h in host_in) * 4)
    out_bytes = int(sum(ho[0].numel() for ho in host_out) * 4)
    c0 = step_counters[0]
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "images/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "latency_s": round(ms / 1e3, 6),
        "higher_is_better": True,
        "scaling": "strong" if groups or W["preset"].channels > 1 else "weak",
        "vs_baseline": None,
        "dtype": "u32",
        "data": "synthetic",
        "config": {
            "workload": W["desc"],
            "model": f"{W['spec'].name}, dense random 4-bit weights (every tap executes)",
            "global_batch": images,
            "parallelism": ("single" if world == 1 else f"output-channel-groups/{world}" if groups
                            else f"replicas{world}" if W["preset"].channels == 1
                            else f"crt-channels/{world}" + (f" + output-channel split of channels "
                                                            f"{[u.channel for u, _ in W['splits']]} over "
                                                            f"{[len(r) for _, r in W['splits']]} ranks"
                                                            if W["splits"] else "")),
            "step": "evaluation of every unit + GPU decryption of the logits on the owning GPU + NCCL gather of "
                    "the plaintext residues to rank 0 + GPU CRT recombination there",
            "units_on_rank0": len(units),
            "crt_channels": len(W["moduli"]),
            **({"groups_on_rank0": D.group_plan(D.groupable(W["spec"]), world)[0]} if groups else {}),
            "hsquare_per_unit": c0.hsquare,
            "mult_plain_per_unit": c0.mult_plain_scheduled,
            "l2_policy": "inputs per GPU >= 565 MB > 126 MB L2 (no flush needed)",
            "setup_s": round(W["setup_s"], 2),
        },
        "e2e": {"value": round(images / (e2e_ms / 1e3), 2), "unit": "images/s",
                "ms_per_step": round(e2e_ms, 3), "wall_ms_per_step": round(wall_e2e * 1e3, 3),
                "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": out_bytes,
                "path": ("pinned host u32 ciphertexts -> distributed.eval_network_groups (every rank uploads the batch) -> "
                         "pinned host logits on rank 0") if groups else
                        "pinned host u32 ciphertexts -> engine.eval_network_stream (upload of step s+1 overlaps "
                        "evaluation of step s; two device input buffers; the first batch streamed by row bands into "
                        "a conv1/square1/conv2/square2 wavefront) -> pinned host logits", "steps": e2e_steps},
        "e2e_dropin": dropin,
        "logits_shape_per_batch": result_shape,
        "gpu_launches": int(launches),
        "host_issue_ms_per_step": round(host_issue_ms, 3),
        "kernels": kernels,
        "roofline": roof,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_cpu_baseline and args.workload == "mnist":
        line["cpu_baseline"] = cpu_baseline_sample(units[0], args.seed, threads=1)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- CPU arms
#
# The reference itself (hefir, installed unmodified into baseline/_ref with
# `pip install --target`; gmpy2 is absent from this image and is replaced by
# tests/_shim/gmpy2.py, `mpz = int`: the same exact integers, slower big-int
# multiplies) is timed on the host cores through its own public API on a
# bounded sample of the MNIST set-1 step, and extrapolated to the full batch:
#   conv     engine.eval_conv on a 7x7 crop of the input -> 2x2x5 = 20 outputs
#            (25 taps each, the dense random weights of the workload); conv1
#            has 720 and conv2 800 such 25-tap outputs (x 1520 / 20)
#   square   engine.eval_square of one ciphertext per host process, `cores`
#            processes at once (x 1520 / cores)
#   fc       engine.eval_fc of one 800-tap output (x 10)
# When baseline/_ref is absent, the pinned oracle port (oracle/) is timed
# the same way instead (kind "port").

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_REF = {}


def _import_hefir():
    if not os.path.isdir(os.path.join(REF_DIR, "hefir")):
        return None
    for p in (os.path.join(ROOT, "tests", "_shim"), REF_DIR):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    try:
        from hefir import bfv, engine, nn_oracle, presets, ring  # noqa: F401
    except Exception:
        return None
    import hefir

    return hefir


def _ref_setup(seed: int):
    """hefir params / keys / one encrypted ciphertext at set 1, and the
    workload's dense random weights (bench.build_workload's seeds)."""
    from hefir import bfv, engine, nn_oracle, presets
    from paper_1811_00778_b200 import nn

    params = presets.build_context(presets.load_preset("1"))
    n = params.ring_degree
    sk, pk, rlk = bfv.keygen(params, np.random.default_rng(seed))
    erng = np.random.default_rng(seed + 5)
    c = bfv.encrypt(pk, bfv.Plaintext(erng.integers(0, MNIST_T, n), MNIST_T), params, erng)
    model = nn.random_model(nn.mnist_hcnn(), np.random.default_rng(seed + 1))
    spec = nn_oracle.mnist_hcnn()
    crop = engine.CipherTensor(shape=(7, 7, 1), cts=[c] * 49, delta=4, channel_modulus=MNIST_T)
    flat = engine.CipherTensor(shape=(1, 1, 800), cts=[c] * 800, delta=4, channel_modulus=MNIST_T)
    one = engine.CipherTensor(shape=(1, 1, 1), cts=[c], delta=4, channel_modulus=MNIST_T)
    _REF.update(params=params, rlk=rlk, crop=crop, flat=flat, one=one, conv1=spec.layers[0], fc=spec.layers[4],
                w_conv=np.asarray(model.weights[0]), w_fc=np.asarray(model.weights[4])[:1], engine=engine)


def _ref_square_worker(_):
    e = _REF["engine"]
    t0 = time.perf_counter()
    e.eval_square(_REF["one"], _REF["rlk"], _REF["params"], e.OpCounter())
    return time.perf_counter() - t0


def _ref_step(cores: int, pool):
    """One bounded sample; returns (seconds of each part)."""
    e, params = _REF["engine"], _REF["params"]
    t0 = time.perf_counter()
    out = e.eval_conv(_REF["crop"], _REF["conv1"], _REF["w_conv"], params, e.OpCounter(), workers=cores)
    t1 = time.perf_counter()
    assert len(out.cts) == 20
    if pool is None:
        _ref_square_worker(0)
    else:
        pool.map(_ref_square_worker, range(cores), chunksize=1)
    t2 = time.perf_counter()
    e.eval_fc(_REF["flat"], _REF["fc"], _REF["w_fc"], params, e.OpCounter(), workers=cores)
    t3 = time.perf_counter()
    return t1 - t0, t2 - t1, t3 - t2


def _extrapolate(t_conv20, t_sq_wall, t_fc1, cores):
    # MNIST step: 720 + 800 25-tap conv outputs, 1520 HSquares, 10 x 800-tap fc outputs
    return (720 + 800) / 20 * t_conv20 + 1520 / cores * t_sq_wall + 10 * t_fc1


def _sample_desc(cores, parts, kind):
    c, q, f = parts
    what = ("hefir (the reference, baseline/_ref, unmodified; gmpy2 shimmed by mpz = int: exact, slower "
            "big-int multiplies than real gmpy2)") if kind == "reference" else "oracle port (oracle/hcnn_oracle.py)"
    return (f"{what} at N=8192/set 1, its public engine API: eval_conv of 20 conv1 outputs ({c:.2f}s), "
            f"eval_square of {cores} ciphertexts on {cores} processes ({q:.2f}s wall), eval_fc of one 800-tap "
            f"output ({f:.2f}s); extrapolated x76 conv, x{1520 / cores:.0f} square, x10 fc to the 8192-image batch")


def _port_step(W, cores):
    """oracle-port fallback: same sample shape"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import hcnn_oracle as O

    params = W["params"]
    op = O.Params(O.Context(params.ring_degree, [pm.value for pm in params.ctx.primes]), params.t)
    rlk = [(k0.residues, k1.residues) for k0, k1 in W["rlk"].components]
    x = W["gin"].data[:1].cpu().numpy().view(np.uint32).astype(np.int64)[0]
    ct = (x[0], x[1])
    t0 = time.perf_counter()
    for _ in range(20):
        O.weighted_sum(op, [(ct, 3)] * 25, O.Counter())
    t1 = time.perf_counter()
    O.hsquare(op, ct, rlk)
    t2 = time.perf_counter()
    O.weighted_sum(op, [(ct, 3)] * 800, O.Counter())
    t3 = time.perf_counter()
    return t1 - t0, t2 - t1, t3 - t2


def cpu_baseline_sample(W, seed: int, threads: int = 1):
    """Our arm's cpu_baseline: one bounded sample of the reference on 1 core."""
    if _import_hefir() is not None:
        _ref_setup(seed)
        parts = _ref_step(1, None)
        kind = "reference"
    else:
        parts = _port_step(W, 1)
        kind = "port"
    T = _extrapolate(*parts, 1)
    return {"value": round(8192 / T, 4), "unit": "images/s", "cores": threads, "kind": kind,
            "latency_s_extrapolated": round(T, 1), "sample": _sample_desc(1, parts, kind)}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp

    cores = os.cpu_count() or 1
    if _import_hefir() is None:
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref (pip install --target of the reference) "
                                                             "is missing or does not import"}), flush=True)
        return
    _ref_setup(args.seed)
    vals, walls = [], []
    with mp.get_context("fork").Pool(cores) as pool:
        for i in range(args.warmup + args.steps):
            w0 = time.perf_counter()
            parts = _ref_step(cores, pool)
            if i >= args.warmup:
                vals.append(parts)
                walls.append(time.perf_counter() - w0)
    parts = tuple(float(np.mean([v[k] for v in vals])) for k in range(3))
    T = _extrapolate(*parts, cores)
    value = 8192 / T
    # ms_per_step is what one timed step (a bounded sample of the batch) took
    # on the host clock; the batch latency the sample extrapolates to is
    # extrapolated_latency_s (value = 8192 images / that latency)
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(float(np.mean(walls)) * 1e3, 1),
        "extrapolated_latency_s": round(T, 2), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int (Python big int / int64)", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": "MNIST HCNN, preset 1 (N=8192, 11 primes, t=5522259017729), one 8192-image slot-batch, "
                               "dense random 4-bit weights",
                   "parallelism": f"{cores} host processes (squares) / eval_conv and eval_fc with workers={cores}"},
        "cpu_baseline": {"value": round(value, 4), "unit": "images/s", "cores": cores, "kind": "reference",
                         "sample": _sample_desc(cores, parts, "reference") + "; per step, mean of the timed steps"},
        "e2e": {"value": round(value, 4), "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the reference with real gmpy2 would multiply faster (its README quotes ~0.29 s per HSquare); "
                "gmpy2 is not installable here",
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
