import os
import sys, time, json
sys.argv = ["bench.py"]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1811_00778_b200 import engine as E
torch.cuda.set_device(0)
W = bench.build_workload("mnist", 0, 1, 2024)
u = W["units"][0]
def step():
    return E.eval_network(u["gin"], u["model"], u["rlk"], u["params"], E.OpCounter())
for _ in range(3): step()
torch.cuda.synchronize()
def timed(k):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k): step()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k
base = timed(5)
h = torch.empty(u["gin"].data.shape, dtype=torch.int32, pin_memory=True)
d = torch.empty_like(u["gin"].data)
cs = torch.cuda.Stream()
with torch.cuda.stream(cs):
    for _ in range(12): d.copy_(h, non_blocking=True)
busy = timed(5)
torch.cuda.synchronize()
# copy alone
t0 = time.perf_counter()
with torch.cuda.stream(cs):
    for _ in range(5): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
print(json.dumps({"step_ms": round(base, 3), "step_ms_with_h2d": round(busy, 3), "h2d_ms": round((time.perf_counter()-t0)*1e3/5, 3)}))
