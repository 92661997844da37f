#!/usr/bin/env python3
"""Timeline of one drop-in engine.eval_network call on a host CipherTensor
(MNIST set 1, 784 ciphertexts): host time of each band's narrowing, and
device time at which each band's upload and wavefront launches complete.

    python tools/dropin_probe.py [--bands 6] [--calls 4]
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

import bench  # noqa: E402
from paper_1811_00778_b200 import engine as E  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bands", type=int, default=6)
    ap.add_argument("--calls", type=int, default=4)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    W = bench.build_workload("mnist", 0, 1, 2024)
    u = W["units"][0]
    hc = u["gin"].to_host()
    E.eval_network(hc, u["model"], u["rlk"], u["params"], E.OpCounter())
    torch.cuda.synchronize()
    st = E._stager(E.context_for(u["params"]))
    orig_fill = st.fill
    marks = []
    t_origin = [0.0]
    ev0 = torch.cuda.Event(enable_timing=True)

    def fill(stage, cts, lo, hi):
        t0 = time.perf_counter()
        orig_fill(stage, cts, lo, hi)
        t1 = time.perf_counter()
        e = torch.cuda.Event(enable_timing=True)
        e.record(torch.cuda.current_stream())  # compute stream: previous band's launches done
        marks.append({"lo": lo, "hi": hi, "host_fill_start_ms": (t0 - t_origin[0]) * 1e3,
                      "host_fill_ms": (t1 - t0) * 1e3, "ev": e})

    st.fill = fill
    for call in range(a.calls):
        marks.clear()
        torch.cuda.synchronize()
        t_origin[0] = time.perf_counter()
        ev0.record()
        out = E._eval_network_host(hc, u["model"], u["rlk"], u["params"], E.OpCounter(), bands=a.bands)
        t_end = time.perf_counter()
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record()
        torch.cuda.synchronize()
        rows = []
        for m in marks:
            rows.append({k: (round(v, 3) if isinstance(v, float) else v) for k, v in m.items() if k != "ev"}
                        | {"device_prev_band_done_ms": round(ev0.elapsed_time(m["ev"]), 3)})
        print(json.dumps({"call": call, "bands": a.bands, "host_total_ms": round((t_end - t_origin[0]) * 1e3, 3),
                          "device_total_ms": round(ev0.elapsed_time(ev1), 3), "bands_detail": rows}))
        del out
    st.fill = orig_fill
    g = E.context_for(u["params"])
    for name, fn in (("dropin", lambda: E._eval_network_host(hc, u["model"], u["rlk"], u["params"], E.OpCounter(),
                                                            bands=a.bands)),
                     ("device", lambda: E.eval_network(u["gin"], u["model"], u["rlk"], u["params"], E.OpCounter()))):
        torch.cuda.synchronize()
        g.profile(True)
        fn()
        torch.cuda.synchronize()
        prof = g.profile_read()
        g.profile(False)
        print(json.dumps({"profile": name, "kernels": {k: [c, round(t, 3)] for k, (c, t) in prof.items()},
                          "total_ms": round(sum(t for _, t in prof.values()), 3)}))


if __name__ == "__main__":
    main()
