"""Host->device copy bandwidth from pinned memory, with and without binding
the process to the CPU cores NVML reports as local to the GPU (the pinned
pages are first-touched by the binding thread, so they land on that node)."""

import json
import os
import sys
import time

import torch


def gpu_local_cpus(dev: int):
    import pynvml

    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(dev)
    words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
    cpus = [w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
    return [c for c in cpus if c < os.cpu_count()]


def measure(nbytes: int, reps: int = 5):
    host = torch.empty(nbytes // 4, dtype=torch.int32, pin_memory=True)
    host.fill_(1)
    dev = torch.empty_like(host, device="cuda")
    dev.copy_(host, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dev.copy_(host, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    return nbytes * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9


if __name__ == "__main__":
    nbytes = int(sys.argv[1]) if len(sys.argv) > 1 else 565182464
    out = {"cpus": os.cpu_count(), "affinity_before": len(os.sched_getaffinity(0))}
    out["h2d_gbs_default"] = round(measure(nbytes), 1)
    local = gpu_local_cpus(0)
    out["gpu_local_cpus"] = f"{local[0]}-{local[-1]} ({len(local)})" if local else None
    if local:
        os.sched_setaffinity(0, local)
        out["h2d_gbs_bound"] = round(measure(nbytes), 1)
    print(json.dumps(out))


def series(nbytes: int, reps: int = 40):
    """GB/s of each of `reps` back-to-back copies of one pinned buffer."""
    host = torch.empty(nbytes // 4, dtype=torch.int32, pin_memory=True)
    host.fill_(1)
    dev = torch.empty_like(host, device="cuda")
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    evs[0].record()
    for i in range(reps):
        dev.copy_(host, non_blocking=True)
        evs[i + 1].record()
    torch.cuda.synchronize()
    return [round(nbytes / (a.elapsed_time(b) * 1e-3) / 1e9, 1) for a, b in zip(evs, evs[1:])]
