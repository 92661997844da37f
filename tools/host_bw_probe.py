#!/usr/bin/env python3
"""Host-side staging probe for the drop-in path (engine._HostStager): the
throughput of hcnn_host_narrow (int64 residue arrays -> pinned u32) by
thread count, plain memcpy bandwidth, pinned H2D bandwidth, and the
fill / upload phases of one MNIST set-1 input (784 ciphertexts).

    python tools/host_bw_probe.py [--out gpurun_out/host_bw.jsonl]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1811_00778_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    n, K, N = 784, 11, 8192
    rng = np.random.default_rng(0)
    arrs = [rng.integers(0, 1 << 30, (K, N)).astype(np.int64) for _ in range(2 * n)]
    ptrs = np.array([x.ctypes.data for x in arrs], dtype=np.uintp)
    dst = torch.empty((2 * n, K, N), dtype=torch.int32, pin_memory=True)
    L = _lib.lib()
    rows = []
    gb_read = 2 * n * K * N * 8 / 1e9
    for threads in (1, 2, 4, 8, 12, 16, 24, 32):
        best = 1e9
        for _ in range(4):
            t0 = time.perf_counter()
            _lib.check(L.hcnn_host_narrow(ptrs.ctypes.data, 2 * n, K * N, _lib.C.c_void_p(dst.data_ptr()), threads))
            best = min(best, time.perf_counter() - t0)
        rows.append({"probe": "host_narrow", "threads": threads, "ms": round(best * 1e3, 2),
                     "gb_read_s": round(gb_read / best, 1)})
    big = np.concatenate([x.reshape(-1) for x in arrs[:n]])
    out = np.empty_like(big)
    t0 = time.perf_counter()
    np.copyto(out, big)
    dt = time.perf_counter() - t0
    rows.append({"probe": "numpy_memcpy_1thread", "gb": round(big.nbytes / 1e9, 3), "gb_s": round(big.nbytes / dt / 1e9, 1)})
    if torch.cuda.is_available():
        d = torch.empty_like(dst, device="cuda")
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            d.copy_(dst, non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        rows.append({"probe": "h2d_pinned", "gb": round(dst.numel() * 4 / 1e9, 3),
                     "gb_s": round(dst.numel() * 4 / dt / 1e9, 1)})
        # narrowing concurrent with the H2D of a previous buffer (both use host memory)
        d2 = torch.empty_like(dst)
        d2 = d2.pin_memory()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d.copy_(d2, non_blocking=True)
        _lib.check(L.hcnn_host_narrow(ptrs.ctypes.data, 2 * n, K * N, _lib.C.c_void_p(dst.data_ptr()), 16))
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rows.append({"probe": "narrow16_during_h2d", "narrow_ms": round((t1 - t0) * 1e3, 2),
                     "both_ms": round((t2 - t0) * 1e3, 2)})
    for r in rows:
        print(json.dumps(r))
    if a.out:
        with open(a.out, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
