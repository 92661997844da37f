#!/usr/bin/env python3
"""Per-primitive latencies on 1 B200: the GPU counterpart of the reference's
`hefir bench` (cli.py:329-387, run_benchmarks) and of the paper's primitive
table (KeyGen, Enc, Dec, HAdd, HMultPlain, HSquare, HMult).

For each preset one JSON line: per primitive
  latency_ms      one operation on one ciphertext (mean of `iters` after 3
                  warm-ups; device ops timed with CUDA events around the call,
                  host-involving ops -- KeyGen / Enc draw their randomness on
                  the host like the reference -- with a wall clock)
  batch_us_per_ct the same device op over `batch` ciphertexts, per ciphertext
HMultPlain uses a full random plaintext polynomial (the reference's general
NTT path).  The reference's ordering check HMultPlain < HSquare <= HMult is
reported as `ordering_ok`.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# the paper's V100 (A*FV) and SEAL CPU numbers, ms
PAPER = {
    "2": {"KeyGen": (12.377, 272.142), "Enc": (0.935, 12.858), "Dec": (0.075, 5.171), "HAdd": (0.052, 0.126),
          "HMultPlain": (0.033, 7.680), "HSquare": (1.679, 69.588), "HMult": (2.014, 86.270)},
    "4": {"KeyGen": (21.392, 542.920), "Enc": (1.496, 25.991), "Dec": (0.098, 10.408), "HAdd": (0.054, 0.281),
          "HMultPlain": (0.035, 15.694), "HSquare": (2.371, 138.199), "HMult": (2.769, 173.167)},
}


def main():
    import torch

    from paper_1811_00778_b200 import bfv as B
    from paper_1811_00778_b200 import engine as E
    from paper_1811_00778_b200 import ops, presets

    ap = argparse.ArgumentParser()
    ap.add_argument("--presets", default="1,2,3,4")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--seed", type=int, default=5)
    a = ap.parse_args()
    torch.cuda.set_device(0)

    def dev_time(fn, iters):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    def wall_time(fn, iters):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(iters):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3 / iters

    for pid in a.presets.split(","):
        preset = presets.load_preset(pid)
        params = presets.build_context(preset, 0)
        rng = np.random.default_rng(a.seed)
        g = E.context_for(params)
        sk, pk, rlk = E.keygen_device(params, rng)
        n = params.ring_degree
        pt = rng.integers(0, params.t, (1, n))
        weight = rng.integers(0, params.t, n)
        centered = np.where(weight > params.t // 2, weight - params.t, weight)
        c1 = E.encrypt_device(pk, pt, params, rng)
        c2 = E.encrypt_device(pk, pt, params, rng)
        big = E.encrypt_device(pk, np.repeat(pt, a.batch, axis=0), params, rng)
        big2 = E.encrypt_device(pk, np.repeat(pt, a.batch, axis=0), params, rng)
        t1 = E.GpuCipherTensor((1, 1, 1), c1, 1, params.t, params)
        tb = E.GpuCipherTensor((1, 1, a.batch), big, 1, params.t, params)
        g.set_relin_key(rlk)
        res = {}
        res["KeyGen"] = (wall_time(lambda: E.keygen_device(params, rng), max(3, a.iters // 4)), None)
        res["Enc"] = (wall_time(lambda: E.encrypt_device(pk, pt, params, rng), a.iters),
                      wall_time(lambda: E.encrypt_device(pk, np.repeat(pt, a.batch, axis=0), params, rng), 3)
                      * 1e3 / a.batch)
        res["Dec"] = (dev_time(lambda: E.decrypt_device(t1, sk, params), a.iters),
                      dev_time(lambda: E.decrypt_device(tb, sk, params), 5) * 1e3 / a.batch)
        res["HAdd"] = (dev_time(lambda: ops.hadd_device(g, c1, c2), a.iters),
                       dev_time(lambda: ops.hadd_device(g, big, big2), 5) * 1e3 / a.batch)
        res["HMultPlain"] = (dev_time(lambda: ops.mul_plain_device(g, c1, centered), a.iters),
                             dev_time(lambda: ops.mul_plain_device(g, big, centered), 5) * 1e3 / a.batch)
        res["HSquare"] = (dev_time(lambda: ops.square_device(g, c1, rlk), a.iters),
                          dev_time(lambda: ops.square_device(g, big, rlk), 5) * 1e3 / a.batch)
        res["HMult"] = (dev_time(lambda: ops.hmult_device(g, c1, c2, rlk), a.iters),
                        dev_time(lambda: ops.hmult_device(g, big, big2, rlk), 5) * 1e3 / a.batch)
        line = {"preset": pid, "n": n, "primes": len(params.ctx.primes), "t": params.t, "batch": a.batch,
                "unit": "ms (latency), us (batch per ct)",
                "primitives": {k: {"latency_ms": round(v[0], 4),
                                   "batch_us_per_ct": None if v[1] is None else round(v[1], 3)}
                               for k, v in res.items()},
                "ordering_ok": res["HMultPlain"][0] < res["HSquare"][0] <= res["HMult"][0] * 1.02,
                "note": "KeyGen and Enc include the host RNG draws (reference order); Dec and the "
                        "evaluation ops are device-timed"}
        if pid in PAPER:
            line["paper_v100_ms"] = {k: v[0] for k, v in PAPER[pid].items()}
            line["paper_seal_cpu_ms"] = {k: v[1] for k, v in PAPER[pid].items()}
        print(json.dumps(line), flush=True)
        del big, big2, tb
        E._CTXS.clear()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
