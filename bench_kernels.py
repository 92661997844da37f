#!/usr/bin/env python3
"""Kernel microbenchmark (BASELINE.json config 2): RNS NTT/INTT and ct x ct
multiply + relinearise over N = 2^13..2^15 and RNS limb counts, on 1 B200.

Each line is one JSON object: per-kernel CUDA-event times (hcnn_profile) and
achieved rates.  Primes: the reference pool (= 1 mod 2^15) for N <= 2^14 and
primes = 1 mod 2^16 below 2^30 for N = 2^15 (the pool does not qualify).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

POOL = (1073643521, 1073479681, 1073184769, 1073053697, 1072857089, 1072496641,
        1071513601, 1071415297, 1071087617, 1070727169, 1070432257, 1069219841)


def primes_1mod(two_n: int, count: int, avoid=()):
    from paper_1811_00778_b200.bfv import is_prime

    out, k = [], 1
    while len(out) < count:
        p = (1 << 30) - k * two_n + 1
        k += 1
        if p not in avoid and is_prime(p):
            out.append(p)
    return out


def _lib_query(g, what):
    from paper_1811_00778_b200 import _lib

    return _lib.lib().hcnn_ctx_query(g.handle, what)


def main():
    import torch

    from paper_1811_00778_b200 import bfv as B
    from paper_1811_00778_b200 import engine as E
    from paper_1811_00778_b200 import ops

    ap = argparse.ArgumentParser()
    ap.add_argument("--ns", default="8192,16384,32768")
    ap.add_argument("--ks", default="6,11,12")
    ap.add_argument("--cts", type=int, default=128)
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--variants", default="default",
                    help="comma list of hcnn_ctx_set_option NTT flags; 'default' = the library's per-N choice")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ntt64", action="store_true",
                    help="u64 NTT rows (62-bit primes, hcnn_ntt64) instead of the u32 sweep")
    a = ap.parse_args()
    if a.ntt64:
        return ntt64_rows(a)
    t = 5522259017729
    for n in [int(x) for x in a.ns.split(",")]:
        for k in [int(x) for x in a.ks.split(",")]:
            primes = list(POOL[:k]) if n <= 16384 else primes_1mod(2 * n, k)
            tt = t if (t - 1) % (2 * n) == 0 else 65537 if n <= 32768 else 65537
            params = B.BfvParams(B.RnsContext(n, primes), tt)
            for variant in a.variants.split(","):
                if variant == "default":
                    os.environ.pop("HCNN_NTT_VARIANT", None)
                else:
                    os.environ["HCNN_NTT_VARIANT"] = str(int(variant))
                E._CTXS.clear()
                g = E.context_for(params)
                sk, pk, rlk = B.keygen(params, np.random.default_rng(1))
                rng = np.random.default_rng(2)
                x = torch.from_numpy(
                    np.stack([np.stack([rng.integers(0, p, n) for p in primes]) for _ in range(2 * a.cts)])
                    .reshape(a.cts, 2, k, n).astype(np.uint32).view(np.int32)).cuda()
                rows = torch.from_numpy(
                    np.stack([rng.integers(0, primes[i % k], n) for i in range(a.rows)]).astype(np.uint32).view(np.int32)).cuda()
                ops.square_device(g, x, rlk)  # warm-up + key upload
                ops.ntt_device(g, rows, k)
                torch.cuda.synchronize()
                g.profile(True)
                for _ in range(a.reps):
                    ops.ntt_device(g, rows, k)
                    ops.ntt_device(g, rows, k, inverse=True)
                    ops.square_device(g, x, rlk)
                torch.cuda.synchronize()
                prof = g.profile_read()
                g.profile(False)
                logn = n.bit_length() - 1
                bfly = n // 2 * logn
                line = {"n": n, "k": k, "kp": g.KP, "digits": g.D,
                        "variant": int(_lib_query(g, 7)), "cts": a.cts,
                        "ntt_rows": a.rows}
                cnt, tot = prof["k_ntt_rows"]
                per = tot / cnt  # ms per launch (fwd or inv of `rows` rows)
                line["ntt_row_us"] = round(per * 1e3 / a.rows, 4)
                line["ntt_gbfly_s"] = round(a.rows * bfly / (per * 1e-3) / 1e9, 1)
                line["ntt_hbm_gbs"] = round(a.rows * n * 8 / (per * 1e-3) / 1e9, 1)
                hsq = 0.0
                for name in ("k_extend", "k_extend_tc", "k_tensor", "k_scale", "k_scale_tc", "k_relin", "k_rb_fwd", "k_rb_mac", "k_rb_mac_tc", "k_rb_inv"):
                    if name not in prof:  # the per-prime or the R-basis relinearisation
                        continue
                    c_, t_ = prof[name]
                    us = t_ / a.reps / a.cts * 1e3
                    line[name + "_us_per_ct"] = round(us, 3)
                    hsq += us
                line["hsquare_us_per_ct"] = round(hsq, 3)
                line["hsquare_bfly_gs"] = round((5 * (k + g.KP) + (g.D + 2) * k) * bfly / (hsq * 1e-6) / 1e9, 1)
                # general ct x ct multiply + relinearise (bfv.hmult: two extensions,
                # 4 forward + 3 inverse transforms per prime), CUDA events around the calls
                y = torch.roll(x, 1, 0).contiguous()
                ops.hmult_device(g, x, y, rlk)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.reps):
                    ops.hmult_device(g, x, y, rlk)
                e1.record()
                torch.cuda.synchronize()
                line["hmult_us_per_ct"] = round(e0.elapsed_time(e1) / a.reps / a.cts * 1e3, 3)
                print(json.dumps(line), flush=True)


def ntt64_rows(a):
    """u64 NTT rows over a 62-bit prime = 1 mod 2N (hcnn_ntt64): forward and
    inverse time per row, butterflies/s, and the fraction of the measured u64
    Harvey butterfly rate (hcnn_int_peak kind 16)."""
    import ctypes

    import torch

    from paper_1811_00778_b200 import _lib
    from paper_1811_00778_b200.bfv import is_prime

    L = _lib.lib()
    peak = ctypes.c_double()
    _lib.check(L.hcnn_int_peak(0, 16, ctypes.byref(peak)))
    for n in [int(x) for x in a.ns.split(",")]:
        k = ((1 << 62) - 1) // (2 * n)
        while not is_prime(k * 2 * n + 1):
            k -= 1
        p = k * 2 * n + 1
        h = ctypes.c_void_p()
        _lib.check(L.hcnn_codec_create(p, n, 0, ctypes.byref(h)))
        rng = np.random.default_rng(n)
        x = torch.from_numpy(rng.integers(0, p, (a.rows, n), dtype=np.uint64).view(np.int64)).cuda()
        st = torch.cuda.current_stream()
        line = {"kernel": "k_ntt64", "n": n, "prime_bits": p.bit_length(), "rows": a.rows,
                "u64_bfly_peak_gs": round(peak.value / 1e9, 1)}
        for inv in (0, 1):
            call = lambda: _lib.check(L.hcnn_ntt64(h, ctypes.c_void_p(x.data_ptr()), a.rows, inv,
                                                   ctypes.c_void_p(st.cuda_stream)))
            for _ in range(2):
                call()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                call()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            bf = a.rows * (n // 2) * (n.bit_length() - 1)
            tag = "inv" if inv else "fwd"
            line[tag + "_row_us"] = round(ms * 1e3 / a.rows, 4)
            line[tag + "_gbfly_s"] = round(bf / (ms * 1e-3) / 1e9, 1)
            line[tag + "_bfly_frac"] = round(bf / (ms * 1e-3) / peak.value, 4)
            line[tag + "_hbm_gbs"] = round(a.rows * n * 16 / (ms * 1e-3) / 1e9, 1)
        L.hcnn_codec_destroy(h)
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
