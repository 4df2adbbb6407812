"""Dev probe: SGD section time (engine events ev[3]->ev[4]) of the cfg3 step."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import paper_2009_09523_b200 as vnt

w = [784, 4096, 4096, 4096, 4096, 10]
e = vnt.Engine(w, "relu", "softmax-cross-entropy")
e.add_device(1 << 20)
P = vnt.param_count(w)
g = np.random.default_rng(0)
e.set_params(g.standard_normal(P) * 0.01)
B, V = 8192, 64
x = torch.randn(B, 784, device="cuda", dtype=torch.float64)
y = torch.softmax(torch.randn(B, 10, device="cuda", dtype=torch.float64), 1)
sizes, dev = vnt.uniform_mapping(B, V, 1)
ups = []
for s in range(8):
    e.train_step_ptr(x.data_ptr(), y.data_ptr(), B, sizes, dev, 0.01, resident=True)
    if s >= 3:
        ups.append(e.timings()["update_ms"])
ms = float(np.mean(ups))
print(f"VNT_SGD_TR={os.environ.get('VNT_SGD_TR', '64')}: SGD {ms * 1e3:.1f} us/step, "
      f"{P * 40 / (ms / 1e3) / 1e9:.0f} GB/s at 40 B/param")
