"""Pinned host->device copy bandwidth (the e2e upload path), 1 and 2 streams."""
import json
import time

import torch

n = 565182464 // 4
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.int32, device="cuda")
res = {}
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    chunk = n // streams
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    res[f"h2d_gbs_{streams}stream"] = round(n * 4 / dt / 1e9, 2)
torch.cuda.synchronize()
t0 = time.perf_counter()
h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
res["d2h_gbs"] = round(n * 4 / (time.perf_counter() - t0) / 1e9, 2)
import subprocess
res["pcie"] = subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max",
                              "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
print(json.dumps(res))
