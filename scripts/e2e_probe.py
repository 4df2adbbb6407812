"""Diagnostics (GPU box): per-step event time, wall time and host time of the
C-ABI calls for cfg3 with device-resident batches against pinned host batches
with vnt_engine_prefetch — whether the e2e path adds host turnaround.
usage: python scripts/e2e_probe.py"""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_2009_09523_b200 as vnt
w = [784, 4096, 4096, 4096, 4096, 10]; B, V = 8192, 64
eng = vnt.Engine(w, "relu", "softmax-cross-entropy"); eng.add_device(1 << 20)
g = np.random.default_rng(1)
eng.set_params(np.concatenate([g.standard_normal(w[i]*w[i+1])/np.sqrt(w[i]) if k == 0 else np.zeros(w[i+1]) for i in range(len(w)-1) for k in (0, 1)]))
sizes, dev_of = vnt.uniform_mapping(B, V, 1, 1 << 20); nd = np.zeros(V, np.int32)
gen = torch.Generator(device="cuda").manual_seed(11)
T = torch.randn(784, 10, device="cuda", dtype=torch.float64, generator=gen) / 28
xs = [torch.randn(B, 784, device="cuda", dtype=torch.float64, generator=gen) for _ in range(4)]
ys = [torch.softmax(x @ T, 1) for x in xs]
hx = [x.cpu().pin_memory() for x in xs]; hy = [y.cpu().pin_memory() for y in ys]
stream = torch.cuda.ExternalStream(eng.stream_ptr())
def run(mode, n=40):
    tp = ts = 0.0
    if mode != "resident": eng.prefetch_ptr(hx[0].data_ptr(), hy[0].data_ptr(), B, sizes, nd, resident=False)
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream); t0 = time.perf_counter()
    for i in range(n):
        a = time.perf_counter()
        if mode == "prefetch" and i + 1 < n: eng.prefetch_ptr(hx[(i+1)%4].data_ptr(), hy[(i+1)%4].data_ptr(), B, sizes, nd, resident=False)
        b = time.perf_counter()
        if mode == "resident": eng.train_step_ptr(xs[i%4].data_ptr(), ys[i%4].data_ptr(), B, sizes, nd, 0.01, resident=True)
        else: eng.train_step_ptr(hx[i%4].data_ptr(), hy[i%4].data_ptr(), B, sizes, nd, 0.01, resident=False)
        c = time.perf_counter(); tp += b - a; ts += c - b
    e1.record(stream); torch.cuda.synchronize()
    print(f"{mode:9s} event {e0.elapsed_time(e1)/n:.3f} ms/step wall {(time.perf_counter()-t0)*1e3/n:.3f} prefetch-call {tp*1e6/n:.1f} us step-call {ts*1e3/n:.3f} ms")
for m in ["resident", "prefetch", "resident", "prefetch"]: run(m)
eng.close()
