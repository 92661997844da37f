"""Timeline of engine.eval_network_stream (events on the three streams)."""
import json
import os
import sys
import time

sys.argv = ["bench.py"]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_1811_00778_b200 import engine as E

torch.cuda.set_device(0)
W = bench.build_workload("mnist", 0, 1, 2024)
u = W["units"][0]
h = torch.empty(u["gin"].data.shape, dtype=torch.int32, pin_memory=True)
h.copy_(u["gin"].data)
steps = 8
outs = [torch.empty((10, 2, 11, 8192), dtype=torch.int32, pin_memory=True) for _ in range(steps)]
marks = []
orig_eval = E.eval_network


def eval_marked(*a, **k):
    s = torch.cuda.Event(enable_timing=True)
    s.record(torch.cuda.current_stream())
    t_host0 = time.perf_counter()
    r = orig_eval(*a, **k)
    e = torch.cuda.Event(enable_timing=True)
    e.record(torch.cuda.current_stream())
    marks.append((s, e, time.perf_counter() - t_host0))
    return r


E.eval_network = eval_marked
for _ in range(2):
    E.eval_network_stream([h] * 3, u["model"], u["rlk"], u["params"], u["gin"].shape, u["gin"].delta,
                          E.OpCounter(), outputs=outs[:3])
marks.clear()
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True)
t0.record()
w0 = time.perf_counter()
E.eval_network_stream([h] * steps, u["model"], u["rlk"], u["params"], u["gin"].shape, u["gin"].delta,
                      E.OpCounter(), outputs=outs)
t1 = torch.cuda.Event(enable_timing=True)
t1.record()
torch.cuda.synchronize()
wall = time.perf_counter() - w0
rows = [{"start_ms": round(t0.elapsed_time(s), 2), "end_ms": round(t0.elapsed_time(e), 2),
         "host_enqueue_ms": round(hq * 1e3, 2)} for s, e, hq in marks]
print(json.dumps({"total_ms": round(t0.elapsed_time(t1), 2), "wall_ms": round(wall * 1e3, 2), "batches": rows}, indent=0))
