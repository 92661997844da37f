"""GPU side of the multi-GPU path on one B200: the CRT recombination kernel
(exact against the reference's formula, ring.py:276-283 / codec.py:48-50),
the output-channel split of a CIFAR-10 channel at set 5 (all ranks run in
lockstep on one GPU, collectives resolved in memory) against the unsplit
network, and bench.py's multi-rank step (2 processes on the one GPU, gloo
with host staging: every code path but NCCL itself)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

from conftest import ROOT  # noqa: E402

from paper_1811_00778_b200 import bfv as B  # noqa: E402
from paper_1811_00778_b200 import distributed as D  # noqa: E402
from paper_1811_00778_b200 import engine as E  # noqa: E402
from paper_1811_00778_b200 import nn, presets  # noqa: E402
from paper_1811_00778_b200.errors import HefirError  # noqa: E402


def _ref_centered(res_cols, moduli):
    total = 1
    for m in moduli:
        total *= m
    acc = 0
    for r, m in zip(res_cols, moduli):  # ring.crt_combine
        big = total // m
        acc += int(r) * big * pow(big % m, -1, m)
    u = acc % total
    return u if u <= total // 2 else u - total  # codec.from_modular


def _wide_moduli(count=16):
    """pairwise coprime odd moduli just above 2^61 (the kernel's upper range)"""
    import math

    out, c = [], (1 << 61) + 1
    while len(out) < count:
        if all(math.gcd(c, m) == 1 for m in out):
            out.append(c)
        c += 2
    return tuple(out)


@pytest.mark.parametrize("which", ["cifar10", "mnist1", "wide"])
def test_crt_combine_kernel_is_exact(which):
    moduli = {"cifar10": tuple(presets.load_preset("5").plaintext_moduli), "mnist1": (5522259017729,),
              "wide": _wide_moduli()}[which]
    total = 1
    for m in moduli:
        total *= m
    rng = np.random.default_rng(4)
    vals = [0, 1, -1, total // 2, -(total // 2), total // 2 - 1]
    vals += [int.from_bytes(rng.bytes(130), "little") % total - total // 2 for _ in range(500)]
    vals += [int(v) for v in rng.integers(-(1 << 40), 1 << 40, 500)]
    res = torch.tensor([[v % m for v in vals] for m in moduli], dtype=torch.int64)
    got = E.crt_combine_device(res.cuda(), moduli)
    exp = [_ref_centered([v % m for m in moduli], moduli) for v in vals]
    assert [int(g) for g in got] == exp


def test_crt_combine_rejects_out_of_range_residues():
    moduli = presets.load_preset("5").plaintext_moduli
    res = torch.zeros((len(moduli), 4), dtype=torch.int64)
    res[3, 2] = moduli[3]
    with pytest.raises(HefirError):
        E.crt_combine_device(res.cuda(), moduli)


def test_reconstruct_logits_cifar_batch_on_gpu():
    """A full CIFAR batch (10 channels x 10 outputs x 8192 images) recombined
    on the GPU equals the reference's per-value loop (engine.py:494-506)."""
    moduli = presets.load_preset("5").plaintext_moduli
    rng = np.random.default_rng(5)
    res = E.ChannelResult(moduli=tuple(moduli), batch_size=8192)
    mats = {t: rng.integers(0, t, (10, 8192)) for t in moduli}
    for t in moduli:
        res.add(t, mats[t])
    got = E.reconstruct_logits(res, moduli)
    assert got.shape == (8192, 10)
    for b in list(range(0, 8192, 997)) + [8191]:
        for o in range(10):
            assert got[b, o] == _ref_centered([mats[t][o, b] for t in moduli], moduli)


@pytest.mark.parametrize("S", [2, 4])
def test_cifar_channel_output_split_equals_unsplit(S):
    """Preset 5, CRT channel 8 (one of the two channels the 8-GPU plan
    splits): the S-rank output-channel split, run in lockstep on this GPU,
    reproduces the unsplit network's logits limb for limb, and the ranks'
    op counters add up to the unsplit counter."""
    params = presets.build_context(presets.load_preset("5"), 8)
    sk, pk, rlk = B.keygen(params, np.random.default_rng(80))
    model = E.reduce_model(nn.random_model(nn.cifar10_hcnn(), np.random.default_rng(81)), params.t)
    images = list(np.random.default_rng(82).integers(0, 256, (32, 32, 32, 3)))
    gin = E.pack_images_device(images, E.PackingLayout(32, params.ring_degree), None, pk, params,
                               np.random.default_rng(83), delta=255)
    c_full = E.OpCounter()
    full = E.eval_network(gin, model, rlk, params, c_full)
    exp = full.residues()
    del full
    counters = [E.OpCounter() for _ in range(S)]
    out = D.run_split_emulated(gin, model, D.GpuSplitBackend(params, rlk), S, counters)
    assert np.array_equal(out.residues(), exp)
    assert out.delta == D.output_delta(model.spec, 255)
    tot = {k: sum(getattr(c, k) for c in counters) for k in c_full.__dict__}
    assert tot == c_full.__dict__
    vals = D.decrypt_residues(out, sk, params, 32).cpu().numpy()
    assert vals.shape == (10, 32)


@pytest.mark.parametrize("workload", ["mnist", "cifar3"])
def test_bench_two_ranks_on_one_gpu_gloo(workload, tmp_path):
    """bench.py under torchrun with 2 ranks (both on this GPU, gloo with host
    staging): the multi-rank step runs end to end and prints one line.
    MNIST: 2 replicas, logits recombined on rank 0; CIFAR with its first 3
    CRT channels (--channels 3, to fit two processes on one GPU): one whole
    channel per rank and channel 2 split by output channel over both."""
    E.release_memory()  # this process's cached device memory: the two ranks need the GPU
    env = dict(os.environ, HCNN_DIST_BACKEND="gloo")
    extra = ["--workload", "mnist"] if workload == "mnist" else ["--workload", "cifar", "--channels", "3"]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(29611 + (workload != "mnist")), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "1", "--warmup", "1", "--no-cpu-baseline", *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=1200, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["logits_shape_per_batch"] == [d["config"]["global_batch"] // (2 if workload == "mnist" else 1), 10]
