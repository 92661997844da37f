"""Run the bench's end-to-end serving loop (eval_network_stream, pinned host
inputs and outputs) several times in one process and print per-step times of
each repetition, plus a per-step timeline of one repetition (upload done,
evaluation start/end on the compute stream), to find where e2e time goes."""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_00778_b200 import engine as E  # noqa: E402

W = bench.build_workload("mnist", 0, 1, 0)
u = W["units"][0]
h = torch.empty(u["gin"].data.shape, dtype=torch.int32, pin_memory=True)
h.copy_(u["gin"].data)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
bands = int(sys.argv[2]) if len(sys.argv) > 2 else 6
n_out = W["spec"].layers[-1].filters
ho = [torch.empty((n_out,) + tuple(h.shape[1:]), dtype=torch.int32, pin_memory=True) for _ in range(steps)]
stream = torch.cuda.current_stream()


def run(k, marks=None):
    hook = None
    if marks is not None:
        def hook(name, t):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            marks.append((name, ev))
    E.eval_network_stream([h] * k, u["model"], u["rlk"], u["params"], u["gin"].shape, u["gin"].delta,
                          E.OpCounter(), outputs=ho, layer_hook=hook, bands=bands)


run(3)
torch.cuda.synchronize()
import time  # noqa: E402

res = []
for rep in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = []
    e0.record(stream)
    w0 = time.perf_counter()
    run(steps, marks)
    w1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    t = [e0.elapsed_time(ev) for _, ev in marks]
    gaps = sorted(((round(b - a, 2), marks[i + 1][0]) for i, (a, b) in enumerate(zip(t, t[1:]))), reverse=True)[:3]
    res.append({"ms_per_step": round(e0.elapsed_time(e1) / steps, 3), "host_call_ms": round((w1 - w0) * 1e3, 1),
                "first_mark_ms": round(t[0], 2), "largest_gaps": gaps})
for r in res:
    print(json.dumps(r))
marks = []
e0 = torch.cuda.Event(enable_timing=True)
e0.record(stream)
run(steps, marks)
torch.cuda.synchronize()
line = [(n, round(e0.elapsed_time(ev), 2)) for n, ev in marks]
print(json.dumps({"timeline_ms": line}))
