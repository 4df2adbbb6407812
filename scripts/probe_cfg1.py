"""Dev probe: where a cfg1 step's time goes (host vs graph vs kernels)."""
import os
import sys
import time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch
import paper_2009_09523_b200 as vnt

w, B, V = [784, 16, 10], 256, 16
e = vnt.Engine(w, "tanh", "softmax-cross-entropy")
e.add_device(1 << 20)
g = np.random.default_rng(1)
e.set_params(np.concatenate([g.standard_normal(784 * 16) / 28, np.zeros(16),
                             g.standard_normal(160) / 4, np.zeros(10)]))
sizes, dev = vnt.uniform_mapping(B, V, 1)
x = torch.randn(B, 784, device="cuda", dtype=torch.float64)
y = torch.softmax(torch.randn(B, 10, device="cuda", dtype=torch.float64), 1)
for _ in range(20):
    e.train_step_ptr(x.data_ptr(), y.data_ptr(), B, sizes, dev, 0.05, resident=True)
torch.cuda.synchronize()
n = 500
t0 = time.perf_counter()
gpu = 0.0
for _ in range(n):
    e.train_step_ptr(x.data_ptr(), y.data_ptr(), B, sizes, dev, 0.05, resident=True)
    gpu += e.timings()["total_ms"]
t1 = time.perf_counter()
print(f"wall/step {1e6 * (t1 - t0) / n:.1f} us, graph device time/step {1e3 * gpu / n:.1f} us")
t0 = time.perf_counter()
for _ in range(n):
    e.timings()
print(f"timings() call {1e6 * (time.perf_counter() - t0) / n:.1f} us")
t0 = time.perf_counter()
for _ in range(n):
    e.lib.vnt_engine_param_count(e.h)
print(f"bare ctypes call {1e6 * (time.perf_counter() - t0) / n:.1f} us")
ns, nd, pm = e._mapping_args(sizes, dev)
t0 = time.perf_counter()
for _ in range(n):
    e._mapping_args(sizes, dev)
print(f"_mapping_args {1e6 * (time.perf_counter() - t0) / n:.1f} us")
e.close()

# e2e-style: pinned host batches, with and without prefetch
e = vnt.Engine(w, "tanh", "softmax-cross-entropy")
e.add_device(1 << 20)
e.set_params(np.concatenate([g.standard_normal(784 * 16) / 28, np.zeros(16),
                             g.standard_normal(160) / 4, np.zeros(10)]))
hx = [torch.randn(B, 784, dtype=torch.float64).pin_memory() for _ in range(4)]
hy = [torch.softmax(torch.randn(B, 10, dtype=torch.float64), 1).pin_memory() for _ in range(4)]
for pf in (False, True):
    for it in range(2):
        t0 = time.perf_counter()
        if pf:
            e.prefetch_ptr(hx[0].data_ptr(), hy[0].data_ptr(), B, sizes, dev, resident=False)
        for i in range(n):
            if pf and i + 1 < n:
                e.prefetch_ptr(hx[(i + 1) % 4].data_ptr(), hy[(i + 1) % 4].data_ptr(), B, sizes, dev,
                               resident=False)
            e.train_step_ptr(hx[i % 4].data_ptr(), hy[i % 4].data_ptr(), B, sizes, dev, 0.05,
                             resident=False)
        t1 = time.perf_counter()
    print(f"host inputs, prefetch={pf}: wall/step {1e6 * (t1 - t0) / n:.1f} us")
e.close()
