"""Per-layer limb-exact spot checks at the benchmarked CIFAR-10 configuration
(SURVEY.md 8(c) parity method (4)): preset 5 (N = 8192, 10 primes), ALL ten
plaintext-CRT channels t_i, the 11-layer CIFAR HCNN with dense random
weights.  Every layer runs on the GPU; for every layer, sampled outputs are
recomputed by the pinned oracle (oracle/hcnn_oracle.py, the reference's
algorithm) FROM THE GPU'S OWN INPUT TO THAT LAYER and compared limb by limb:

  conv    the 4 corner output positions (padding taps) + 4 random ones
  square  4 random HSquares (exact tensor, t_i/q rounding, relinearisation)
  pool    4 random windows
  fc      fc1: first, last and one random output; fc2: all 10 outputs

The same harness runs the MNIST HCNN at preset 3 (N = 16384).  (Preset 1,
the MNIST bench config, is pinned completely, every limb of every layer, by
test_gpu_parity.test_set1_bench_workload_every_layer_equals_the_reference.)
The oracle work is fanned over forked host processes per channel."""

import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)

import hcnn_oracle as O  # noqa: E402

from paper_1811_00778_b200 import bfv as B  # noqa: E402
from paper_1811_00778_b200 import engine as E  # noqa: E402
from paper_1811_00778_b200 import nn, presets  # noqa: E402
from paper_1811_00778_b200.nn import kind_of  # noqa: E402

_JOBS = {}  # read by the forked workers


def _fetch(t: E.GpuCipherTensor, idx) -> dict:
    idx = sorted(set(int(i) for i in idx))
    sel = t.data.index_select(0, torch.tensor(idx, device=t.data.device))
    arr = sel.cpu().numpy().view(np.uint32).astype(np.int64)
    return {i: (arr[k, 0], arr[k, 1]) for k, i in enumerate(idx)}


def _conv_taps(layer, weights, ishape, oy, ox, f):
    h, w, c = ishape
    _, kh, kw, cg = weights.shape
    sh, sw = layer.stride
    ph = (kh - 1) // 2 if layer.padded else 0
    pw = (kw - 1) // 2 if layer.padded else 0
    per = weights.shape[0] // layer.groups
    g = f // per
    taps = []
    for ky in range(kh):
        iy = oy * sh + ky - ph
        if not 0 <= iy < h:
            continue
        for kx in range(kw):
            ix = ox * sw + kx - pw
            if not 0 <= ix < w:
                continue
            for ci in range(cg):
                taps.append(((iy * w + ix) * c + g * cg + ci, int(weights[f][ky][kx][ci])))
    return taps


def _run_job(i):
    job = _JOBS["jobs"][i]
    op, rlk = _JOBS["op"], _JOBS["rlk"]
    kind = job["kind"]
    if kind == "sum":  # conv / fc output: the reference's weighted sum over the GPU's inputs
        src = job["src"]
        exp = O.weighted_sum(op, [(src[j], wv) for j, wv in job["taps"]], O.Counter())
    elif kind == "square":
        exp = O.hsquare(op, job["src"], rlk)
    else:  # pool window: hadd chain
        cts = job["src"]
        m = op.ctx.mods
        a0, a1 = cts[0]
        for c0, c1 in cts[1:]:
            a0, a1 = (a0 + c0) % m, (a1 + c1) % m
        exp = (a0, a1)
    got = job["got"]
    return bool(np.array_equal(np.stack(exp), np.stack(got))), job["what"]


def _spot_check_network(params, spec, model, gin, rlk, seed):
    """Evaluate on the GPU layer by layer and queue oracle jobs per layer."""
    rng = np.random.default_rng(seed)
    jobs = []
    prev = [gin]

    def hook(name, out):
        x = prev[0]
        layer = next(la for la in spec.layers if la.name == name)
        li = list(spec.layers).index(layer)
        weights = model.weights[li]
        k = kind_of(layer)
        oh, ow, oc = out.shape
        if k == "conv":
            weights = np.asarray(weights)
            pos = [(0, 0), (0, ow - 1), (oh - 1, 0), (oh - 1, ow - 1)]
            pos += [(int(rng.integers(0, oh)), int(rng.integers(0, ow))) for _ in range(4)]
            sel = [(oy, ox, int(rng.integers(0, oc))) for oy, ox in pos]
            taps = [_conv_taps(layer, weights, x.shape, oy, ox, f) for oy, ox, f in sel]
            src = _fetch(x, [j for tp in taps for j, _ in tp])
            outs = _fetch(out, [(oy * ow + ox) * oc + f for oy, ox, f in sel])
            for (oy, ox, f), tp in zip(sel, taps):
                jobs.append(dict(kind="sum", src={j: src[j] for j, _ in tp}, taps=tp,
                                 got=outs[(oy * ow + ox) * oc + f], what=f"{name}[{oy},{ox},{f}]"))
        elif k == "square":
            idx = [int(i) for i in rng.choice(len(out), 4, replace=False)]
            src, outs = _fetch(x, idx), _fetch(out, idx)
            for i in idx:
                jobs.append(dict(kind="square", src=src[i], got=outs[i], what=f"{name}[{i}]"))
        elif k == "pool":
            h, w, c = x.shape
            e = layer.extent
            sh, sw = layer.stride
            for _ in range(4):
                oy, ox, ch = int(rng.integers(0, oh)), int(rng.integers(0, ow)), int(rng.integers(0, oc))
                win = [((oy * sh + dy) * w + ox * sw + dx) * c + ch for dy in range(e) for dx in range(e)]
                src = _fetch(x, win)
                o = (oy * ow + ox) * oc + ch
                jobs.append(dict(kind="pool", src=[src[j] for j in win], got=_fetch(out, [o])[o],
                                 what=f"{name}[{oy},{ox},{ch}]"))
        elif k == "fc":
            weights = np.asarray(weights)
            n_out = weights.shape[0]
            sel = list(range(n_out)) if n_out <= 10 else [0, n_out - 1, int(rng.integers(1, n_out - 1))]
            src = _fetch(x, range(len(x)))
            outs = _fetch(out, sel)
            for o in sel:
                tp = [(j, int(weights[o][j])) for j in range(weights.shape[1])]
                jobs.append(dict(kind="sum", src=src, taps=tp, got=outs[o], what=f"{name}[{o}]"))
        prev[0] = out

    counter = E.OpCounter()
    E.eval_network(gin, model, rlk, params, counter, layer_hook=hook)
    torch.cuda.synchronize()
    return jobs, counter


def _check_jobs(params, rlk, jobs):
    _JOBS.clear()
    _JOBS.update(jobs=jobs, rlk=[(k0.residues, k1.residues) for k0, k1 in rlk.components],
                 op=O.Params(O.Context(params.ring_degree, [pm.value for pm in params.ctx.primes]), params.t))
    with mp.get_context("fork").Pool(min(16, os.cpu_count() or 1)) as pool:
        res = pool.map(_run_job, range(len(jobs)), chunksize=1)
    bad = [what for ok, what in res if not ok]
    assert not bad, f"limb mismatch at {bad}"
    return len(res)


@pytest.mark.parametrize("channel", list(range(10)))
def test_cifar_set5_every_layer_spot_checked_all_channels(channel):
    preset = presets.load_preset("5")
    params = presets.build_context(preset, channel)
    sk, pk, rlk = B.keygen(params, np.random.default_rng(500 + channel))
    spec = nn.cifar10_hcnn()
    model = E.reduce_model(nn.random_model(spec, np.random.default_rng(77)), params.t)
    n = params.ring_degree
    images = list(np.random.default_rng(78).integers(0, 256, (64, 32, 32, 3)))
    gin = E.pack_images_device(images, E.PackingLayout(64, n), None, pk, params,
                               np.random.default_rng(600 + channel), delta=255)
    jobs, counter = _spot_check_network(params, spec, model, gin, rlk, seed=channel)
    assert counter.hsquare == 32768 + 16384 + 8192
    checked = _check_jobs(params, rlk, jobs)
    assert checked == 3 * 8 + 3 * 4 + 3 * 4 + 3 + 10


def test_mnist_set3_every_layer_spot_checked():
    preset = presets.load_preset("3")
    params = presets.build_context(preset, 0)
    sk, pk, rlk = B.keygen(params, np.random.default_rng(31))
    spec = nn.mnist_hcnn()
    model = E.reduce_model(nn.random_model(spec, np.random.default_rng(32)), params.t)
    n = params.ring_degree
    images = list(np.random.default_rng(33).integers(0, 5, (16, 28, 28, 1)))
    gin = E.pack_images_device(images, E.PackingLayout(16, n), None, pk, params, np.random.default_rng(34), delta=4)
    jobs, counter = _spot_check_network(params, spec, model, gin, rlk, seed=3)
    assert counter.hsquare == 720 + 800
    assert _check_jobs(params, rlk, jobs) == 2 * 8 + 2 * 4 + 10
