"""Time the dense layer alone (CIFAR fc1 shape by default: 2048 -> 256 at set 5)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1811_00778_b200 import engine as E
from paper_1811_00778_b200 import nn, presets

ap = argparse.ArgumentParser()
ap.add_argument("--n-in", type=int, default=2048)
ap.add_argument("--n-out", type=int, default=256)
ap.add_argument("--scale", type=int, default=1023)
ap.add_argument("--preset", default="5")
a = ap.parse_args()
params = presets.build_context(presets.load_preset(a.preset), 0)
g = E.context_for(params)
rng = np.random.default_rng(1)
x = torch.randint(0, 1 << 29, (a.n_in, 2, g.K, g.N), dtype=torch.int32, device="cuda")
tin = E.GpuCipherTensor((1, 1, a.n_in), x, 1, params.t, params)
w = rng.integers(-a.scale, a.scale + 1, (a.n_out, a.n_in))
layer = nn.fc_layer("fc", a.n_out, a.scale)
for _ in range(3):
    E.eval_fc(tin, layer, w, params, E.OpCounter())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    E.eval_fc(tin, layer, w, params, E.OpCounter())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
macs = a.n_in * a.n_out * 2 * g.K * g.N
print(json.dumps({"n_in": a.n_in, "n_out": a.n_out, "ms": round(ms, 3), "dfma_tflops": round(2 * macs / ms / 1e9, 2),
                  "input_gb": round(a.n_in * 2 * g.K * g.N * 4 / 1e9, 3)}))
