#!/usr/bin/env python3
"""Per-band timeline of the drop-in engine.eval_network on a host
CipherTensor (MNIST set 1): host time when each band's launches were issued,
device time when its upload and its wavefront kernels completed.

    python tools/dropin_trace.py [--bands 6] [--calls 3]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1811_00778_b200 import engine as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bands", type=int, default=6)
    ap.add_argument("--calls", type=int, default=3)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    W = bench.build_workload("mnist", 0, 1, 2024)
    u = W["units"][0]
    hc = u["gin"].to_host()
    E._eval_network_host(hc, u["model"], u["rlk"], u["params"], E.OpCounter(), bands=a.bands)
    torch.cuda.synchronize()
    marks = {}

    def wrap(name, fn):
        def w(*args, **kw):
            t = time.perf_counter()
            r = fn(*args, **kw)
            marks[name] = (round((t - marks["t0"]) * 1e3, 2), round((time.perf_counter() - t) * 1e3, 2))
            return r
        return w

    E._banded_head = wrap("banded_head", E._banded_head)
    E._eval_layers = wrap("eval_layers", E._eval_layers)
    E.GpuCipherTensor.to_host = wrap("to_host", E.GpuCipherTensor.to_host)
    for call in range(a.calls):
        marks["t0"] = time.perf_counter()
        E._BAND_TRACE = []
        ev0 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev0.record()
        E._eval_network_host(hc, u["model"], u["rlk"], u["params"], E.OpCounter(), bands=a.bands)
        t1 = time.perf_counter()
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record()
        torch.cuda.synchronize()
        rows = [{"cts": n, "host_ms": round((t - t0) * 1e3, 2), "upload_done_ms": round(ev0.elapsed_time(up), 2),
                 "compute_done_ms": round(ev0.elapsed_time(dn), 2)} for n, t, up, dn in E._BAND_TRACE]
        print(json.dumps({"call": call, "bands": a.bands, "host_total_ms": round((t1 - t0) * 1e3, 2),
                          "device_total_ms": round(ev0.elapsed_time(ev1), 2),
                          "host_segments_start_dur_ms": {k: v for k, v in marks.items() if k != "t0"},
                          "trace": rows}))
    E._BAND_TRACE = None


if __name__ == "__main__":
    main()
