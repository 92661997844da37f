"""Host-side cost of one MNIST step: wall time to ENQUEUE k eval_network calls
(no synchronisation) against their device time, plus a cProfile of the
enqueue loop.  If enqueue wall ~ device time, something in the host path
blocks on the GPU."""

import cProfile
import json
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1811_00778_b200 import engine as E  # noqa: E402

W = bench.build_workload(sys.argv[1] if len(sys.argv) > 1 else "mnist", 0, 1, 0)
u = W["units"][0]
for _ in range(3):
    E.eval_network(u["gin"], u["model"], u["rlk"], u["params"], E.OpCounter())
torch.cuda.synchronize()
k = 10
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
w0 = time.perf_counter()
for _ in range(k):
    E.eval_network(u["gin"], u["model"], u["rlk"], u["params"], E.OpCounter())
w1 = time.perf_counter()
e1.record()
torch.cuda.synchronize()
out = {"enqueue_ms_per_step": round((w1 - w0) * 1e3 / k, 3), "device_ms_per_step": round(e0.elapsed_time(e1) / k, 3)}
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    E.eval_network(u["gin"], u["model"], u["rlk"], u["params"], E.OpCounter())
pr.disable()
torch.cuda.synchronize()
print(json.dumps(out))
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
