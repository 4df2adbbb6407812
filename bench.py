#!/usr/bin/env python
"""Virtual-node training-step benchmark (BASELINE.json metric: samples/sec at
fixed global batch and V).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3]
                    [--impl ours|reference] [--gemm-mode auto]

A "step" is one Trainer::step of the hot path (runner.cpp:75-82): forward +
backward of every virtual node, exact gradient reduction (NCCL all-reduce when
N > 1), fused SGD.  Default workload = BASELINE config 3 (wide MLP
[784,4096x4,10] relu/softmax-CE fp32, B = 8192, V = 64), the GEMM-bound
configuration the north star's roofline target is stated on.  N > 1: launch
with torch.distributed.run, one rank per GPU; virtual nodes are dealt
round-robin (make_uniform_mapping) so per-GPU work is B/N (fixed global batch).

One JSON line on rank 0.  `value` = samples/s with the batch resident in HBM;
`e2e` = the same through the C-ABI with pinned host batches (H2D + loss D2H in
the timed region).  `--impl reference` times the reference's own CPU
implementation (oracle/_ref, else our C port) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: widths, act, loss, B, V, lr, capacity
    "cfg1": dict(widths=[784, 16, 10], act="tanh", loss="softmax-cross-entropy", B=256, V=16,
                 lr=0.05, capacity=1 << 20, config_index=1),
    "cfg3": dict(widths=[784, 4096, 4096, 4096, 4096, 10], act="relu",
                 loss="softmax-cross-entropy", B=8192, V=64, lr=0.01, capacity=1 << 20,
                 config_index=2),
    "cfg4": dict(widths=[784, 4096, 4096, 4096, 4096, 10], act="relu",
                 loss="softmax-cross-entropy", B=65536, V=256, lr=0.01, capacity=256,
                 config_index=3),
}


def gemm_flops_per_step(widths, B):
    """B * 2 * (3*sum_ww - w0*w1) (fwd + bwd-data except layer 0 + dW)."""
    sww = sum(widths[i] * widths[i + 1] for i in range(len(widths) - 1))
    return B * 2 * (3 * sww - widths[0] * widths[1])


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
        "fallback (B200_PROFILING.md)"


def host_cpu():
    """nproc and the CPU model of this host (the reference arm's cores)."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def measure_tf32_peak(seconds=3.0):
    """Sustained dense TF32 tensor throughput of this GPU: cuBLAS TF32 GEMMs at
    8192^3 for `seconds` (the denominator of roofline.frac for the TF32 modes;
    MEASURED_PEAKS.json has no TF32 figure)."""
    import torch
    prev = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    c = torch.empty(n, n, device="cuda")
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters, ms = 0, 0.0
    t0 = time.perf_counter()
    e0.record()
    while time.perf_counter() - t0 < seconds:
        for _ in range(10):
            torch.matmul(a, b, out=c)
        iters += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    torch.backends.cuda.matmul.allow_tf32 = prev
    del a, b, c
    return 2.0 * n ** 3 * iters / (ms / 1e3) / 1e12


def headline_parity(vnt, work):
    """cpu_baseline leg, the CPU path as the checker: the engine's mean gradient
    and loss at the workload's widths (B = 64, V = 8) against the fp64 C port
    of the reference (oracle/, vo_forward_backward_wide; relu masks of
    near-zero pre-activations resolved as tests/test_headline_parity_gpu.py)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    port = oracle_lib.port()
    w, act, loss = work["widths"], work["act"], work["loss"]
    B, V = 64, 8
    p0 = port.init_params(w, 1)
    x, y = port.synth_batch(1, 65536, w[0], w[-1], 0, B)
    e = vnt.Engine(w, act, loss, gemm_mode="auto")
    e.add_device(1 << 20)
    e.set_params(p0)
    e.device_step(0, x, y, np.full(V, B // V, np.uint64))
    acts = {l: e.debug_activation(l, B) for l in range(1, len(w) - 1)} if act == "relu" else None
    g, ls, ex = e.sync()
    e.close()
    g_ref, l_ref, flips, conflicts = port.forward_backward_wide(w, act, loss, p0, x, y, act_ext=acts,
                                                                tau=3e-5, counts=True)
    worst, off = 0.0, 0
    for l in range(len(w) - 1):
        for n in (w[l] * w[l + 1], w[l + 1]):
            m = np.abs(g_ref[off:off + n]).max()
            if m > 0:
                worst = max(worst, float(np.abs(g[off:off + n] - g_ref[off:off + n]).max() / m))
            off += n
    return {"grad_dev_of_max": worst, "loss_rel_dev": abs(ls / ex - l_ref) / abs(l_ref),
            "tolerance": {"grad_dev_of_max": 2e-5, "loss_rel_dev": 2e-6},
            "relu_masks_resolved": flips, "mask_conflicts": conflicts,
            "sample": f"B={B}, V={V}, widths {w}, gemm_mode auto (split-fp16 tcgen05); reference: fp64 C port"}


class ClockSampler:
    """SM clock + throttle reasons sampled during the timed region: NVML polled
    every 2 ms from a thread (a 1-ms cfg1 region still gets samples), else
    nvidia-smi at 25 ms."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0):
        self.index = index
        # NVML and nvidia-smi number GPUs physically; CUDA_VISIBLE_DEVICES may
        # renumber them: address the GPU by its UUID
        self.uuid = None
        try:
            import torch
            self.uuid = "GPU-" + str(torch.cuda.get_device_properties(index).uuid)
        except Exception:
            pass
        self.proc = None
        self.nvml = None
        self.stop = threading.Event()
        self.samples = []      # (sm_mhz, max_mhz, set(reasons))
        self.lines = []

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = (pynvml.nvmlDeviceGetHandleByUUID(self.uuid) if self.uuid
                 else pynvml.nvmlDeviceGetHandleByIndex(self.index))
            bits = {"hw_slowdown": pynvml.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksThrottleReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksThrottleReasonSwPowerCap}
            mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self.stop.is_set():
                    try:
                        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        self.samples.append((sm, mx, {n for n, b in bits.items() if r & b}))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.nvml = pynvml
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.uuid or str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a while to start: a short timed region (20 steps
            # of ~6.5 ms) would otherwise end before its first sample
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
            self.lines.clear()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.nvml is not None:
            self.stop.set()
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        for s_, m_, r_ in self.samples:
            sm.append(s_)
            mx = m_
            reasons |= r_
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi",
                "gpu": self.uuid or self.index}


# ------------------------------------------------------------------ reference arm
def cpu_reference(work, steps, warmup):
    """The reference's own CPU implementation (oracle/_ref), bounded sample.

    cfg1: full Trainer::step (runner.cpp:75-82).  cfg3/cfg4: a full step needs
    two 71-limb exact accumulators of 30 GB each and ~6 h; the sample is
    Model::accumulate_example_grads over a few full-width examples plus one
    ExactVectorAccumulator::rounded(), extrapolated linearly to B examples."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib
    ref = oracle_lib.ref()
    kind = "reference" if ref is not None else "port"
    o = ref if ref is not None else oracle_lib.port()
    w, B, V = work["widths"], work["B"], work["V"]
    cores = 1
    if work["widths"][1] <= 256:
        # full Trainer::step; reference parallelism = one std::async thread per
        # simulated device (parallel_devices, virtual_exec.cpp:242-251): best G.
        best = None
        for G in sorted({1, 2, 4, 8, 16, os.cpu_count() or 1}):
            if G > V or G > (os.cpu_count() or 1):
                continue
            if kind == "reference":
                t = o.trainer(w, work["act"], work["loss"], 11, B, V, work["lr"], 11, 60000, G,
                              parallel=True)
            else:
                t = o.trainer(w, work["act"], work["loss"], 11, B, V, work["lr"], 11, 60000, G)
            for _ in range(warmup):
                t.step()
            t0 = time.perf_counter()
            for _ in range(steps):
                t.step()
            dt = (time.perf_counter() - t0) / steps
            if best is None or dt < best[0]:
                best = (dt, G)
        dt, G = best
        return {"value": B / dt, "unit": "samples/s", "cores": G if kind == "reference" else 1,
                "kind": kind, "sample": f"{steps} full Trainer::step of B={B}, V={V}, "
                f"G={G} devices (parallel_devices={kind == 'reference'}), best of G in 1..16",
                "extrapolated": False, "steps_timed": steps, **host_cpu()}, dt
    # wide model: bounded sample (needs ~31 GB host RAM for the exact accumulator)
    avail = 0
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable"):
                avail = int(ln.split()[1]) * 1024
    except OSError:
        pass
    P = sum(w[i] * w[i + 1] + w[i + 1] for i in range(len(w) - 1))
    need = P * 71 * 8 * 1.15
    n_ex = 2
    x, y = o.synth_batch(1, 65536, w[0], w[-1], 0, n_ex)
    if ref is not None and avail > need:
        import ctypes as C
        wa = (C.c_uint64 * len(w))(*w)
        fp = C.POINTER(C.c_double)
        # one thread per simulated device, each with its own 71-limb accumulator
        threads = int(max(1, min(os.cpu_count() or 1, (avail - 16 * 2**30) // need)))
        f = ref.lib.vntref_accumulate_sample_mt
        wall = C.c_double()
        rc = f(wa, C.c_uint32(len(w)), C.c_int(0), C.c_int(1), C.c_uint64(1),
               x.ctypes.data_as(fp), y.ctypes.data_as(fp), C.c_uint64(n_ex), C.c_uint32(threads),
               C.byref(wall))
        assert rc == 0
        g = ref.lib.vntref_accumulate_sample
        acc_s, rnd_s = C.c_double(), C.c_double()
        rc = g(wa, C.c_uint32(len(w)), C.c_int(0), C.c_int(1), C.c_uint64(1),
               x.ctypes.data_as(fp), y.ctypes.data_as(fp), C.c_uint64(1), C.byref(acc_s),
               C.byref(rnd_s))
        assert rc == 0
        per_ex = wall.value / (n_ex * threads)      # throughput-equivalent per example
        step_s = B * per_ex + rnd_s.value * 2 / threads
        cores = threads
        sample = (f"Model::accumulate_example_grads, {threads} threads x {n_ex} full-width "
                  f"examples each ({wall.value:.1f} s wall, one exact accumulator per thread) + "
                  f"ExactVectorAccumulator::rounded ({rnd_s.value:.1f} s, x2 for device + sync "
                  f"rounding, split over threads), linearly extrapolated to B={B}")
    else:
        kind = "port"
        t0 = time.perf_counter()
        p = oracle_lib.port().init_params(w, 1)
        oracle_lib.port().forward_backward(w, work["act"], work["loss"], p, x, y)
        per = time.perf_counter() - t0
        step_s = B * per / n_ex
        sample = (f"C port forward_backward on {n_ex} full-width examples ({per:.1f} s, "
                  f"MemAvailable {avail/2**30:.0f} GiB < exact-accumulator need), "
                  f"extrapolated to B={B}")
    return {"value": B / step_s, "unit": "samples/s", "cores": cores, "kind": kind,
            "sample": sample, "extrapolated": True, "examples_timed": n_ex * cores, **host_cpu()}, step_s


def run_config(args, work, world):
    """The `config` object both arms print (same workload, same keys)."""
    return {"workload": args.workload, "baseline_config_index": work["config_index"],
            "layer_widths": work["widths"], "activation": work["act"], "loss": work["loss"],
            "global_batch": work["B"], "virtual_nodes": work["V"], "lr": work["lr"],
            "parallelism": f"vn-dp{world}", "gemm_mode": args.gemm_mode,
            "l2": "per-step working set (fp64+fp32 params, activations) >> 126 MB L2; "
                  "4 resident batches rotate"}


def run_reference(args, work):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    base, step_s = cpu_reference(work, max(1, min(args.steps, 3)), 1 if work["widths"][1] <= 256 else 0)
    line = {
        "metric": "samples/sec at fixed global batch & V", "impl": "reference",
        "timed": ("a bounded sample of the step, linearly extrapolated (cpu_baseline.sample); "
                  "steps/warmup below are the requested ones") if base.get("extrapolated") else
                 f"{base.get('steps_timed')} full steps",
        "value": base["value"], "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": run_config(args, work, int(os.environ.get("WORLD_SIZE", "1"))),
        "cpu_baseline": base,
        "e2e": {"value": base["value"], "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ our arm
def run_ours(args, work):
    import torch
    import torch.distributed as dist
    import paper_2009_09523_b200 as vnt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    nccl_id = None
    if world > 1:
        obj = [vnt.Engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    # The timed region runs every step as one CUDA-graph replay (host prep, one
    # graph launch, one synchronize); the GEMM roofline numbers come from a short
    # eager run afterwards with CUDA events around each GEMM launch (events inside
    # graphs cannot be timed).  --eager times the eager, profiled launches instead.
    # (with an NCCL group the engine launches eagerly anyway: profile in place)
    # N > 1: the NCCL collectives are captured with the step (engine.cu).  The
    # GEMM launch times never come from the timed region: a separate eager,
    # profiled single-process engine replays this rank's local nodes afterwards.
    graph_mode = not args.eager
    os.environ["VNT_PROFILE_KERNELS"] = "0" if graph_mode else "1"
    w, B, V, lr = work["widths"], work["B"], work["V"], work["lr"]
    eng = vnt.Engine(w, work["act"], work["loss"], cuda_device=local, rank=rank,
                     world_size=world, nccl_id=nccl_id, gemm_mode=args.gemm_mode,
                     resident_rows=args.resident_rows)
    eng.add_device(work["capacity"])
    g = np.random.default_rng(1)
    params = []
    for i in range(len(w) - 1):
        params.append(g.standard_normal(w[i] * w[i + 1]) / np.sqrt(w[i]))
        params.append(np.zeros(w[i + 1]))
    eng.set_params(np.concatenate(params))
    sizes, dev_of = vnt.uniform_mapping(B, V, world, work["capacity"])
    node_device = np.where(dev_of == rank, 0, -1).astype(np.int32)

    # Synthetic batches of the named shape (SynthDataset semantics, data.cpp:50-105:
    # x ~ N(0,1), soft labels softmax(x T)), resident in HBM, fp64 like vnt::Batch.
    nb = 4
    gen = torch.Generator(device="cuda").manual_seed(11)
    T = torch.randn(w[0], w[-1], device="cuda", dtype=torch.float64, generator=gen) / w[0] ** 0.5
    xs, ys = [], []
    for _ in range(nb):
        x = torch.randn(B, w[0], device="cuda", dtype=torch.float64, generator=gen)
        xs.append(x)
        ys.append(torch.softmax(x @ T, dim=1))
    stream = torch.cuda.ExternalStream(eng.stream_ptr())

    def step(i, resident=True, host=None):
        if resident:
            return eng.train_step_ptr(xs[i % nb].data_ptr(), ys[i % nb].data_ptr(), B, sizes,
                                      node_device, lr, resident=True)
        hx, hy = host
        return eng.train_step_ptr(hx[i % nb].data_ptr(), hy[i % nb].data_ptr(), B, sizes,
                                  node_device, lr, resident=False)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        step(i)
    barrier()
    gemm_ms, gemm_fl, gemm_n, launches = 0.0, 0.0, 0, 0
    with ClockSampler(local) as clocks:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        losses = []
        for i in range(args.steps):
            losses.append(step(i))
            t = eng.timings()
            gemm_ms += t["gemm_ms"]
            gemm_fl += t["gemm_flops"]
            gemm_n += t["gemm_launches"]
            launches += t["kernel_launches"]
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / args.steps
    value = B / (ms_per_step / 1e3)

    # e2e: through the C-ABI with pinned host batches (H2D of the rank's rows +
    # loss/flag D2H inside the timed region).
    hx = [x.cpu().pin_memory() for x in xs]
    hy = [y.cpu().pin_memory() for y in ys]
    def prefetch(i):
        if not args.no_prefetch:
            eng.prefetch_ptr(hx[i % nb].data_ptr(), hy[i % nb].data_ptr(), B, sizes, node_device,
                             resident=False)

    # untimed warm-up of the same prefetch pattern (graphs for both input buffers)
    prefetch(0)
    for i in range(max(args.warmup, 4)):
        prefetch(i + 1)
        step(i, resident=False, host=(hx, hy))
    step(max(args.warmup, 4), resident=False, host=(hx, hy))   # consumes the last prefetch
    barrier()
    t0 = time.perf_counter()
    e0.record(stream)
    # vnt_engine_prefetch: batch i+1's H2D runs on the engine's copy stream
    # while step i computes (runner.cpp:64-73's prefetch, on the device).
    prefetch(0)
    for i in range(args.steps):
        if i + 1 < args.steps:
            prefetch(i + 1)
        step(i, resident=False, host=(hx, hy))
    e1.record(stream)
    barrier()
    e2e_wall_ms = (time.perf_counter() - t0) * 1e3
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = B / (e2e_ms / args.steps / 1e3)
    local_rows = int(sizes[node_device >= 0].sum())
    h2d = local_rows * (w[0] + w[-1]) * 8
    d2h = (3 + 2 * (len(w) - 1)) * 8 + 2 * (len(w) - 1) * 8

    peaks, peak_src = measured_peaks()
    flops_step = gemm_flops_per_step(w, B)
    line = {
        "metric": "samples/sec at fixed global batch & V", "value": value, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "arithmetic": {"auto": "dense GEMMs: fp32 emulated by split-fp16 operands (x 2^s = hi + lo) on tcgen05 "
                               "kind::f16, three MMAs per k16 step, fp32 accumulation; per-node gradients "
                               "int64 fixed point; update fp64",
                       "3xf16": "as auto", "3xtf32": "as auto", "tf32": "dense GEMMs: 1-pass tcgen05 kind::tf32",
                       "ffma": "fp32 FMA everywhere"}[args.gemm_mode],
        "config": run_config(args, work, world),
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "prefetch": not args.no_prefetch,
                "wall_ms_per_step": e2e_wall_ms / args.steps},
        "gpu_launches": launches,
        "final_loss": losses[-1],
        "clocks": clocks.summary(),
    }
    if graph_mode:
        # this rank's nodes (all of them at N = 1) on a world-1 engine, eager,
        # CUDA events around each GEMM launch
        os.environ["VNT_PROFILE_KERNELS"] = "1"
        pe = vnt.Engine(w, work["act"], work["loss"], cuda_device=local, gemm_mode=args.gemm_mode,
                        resident_rows=args.resident_rows)
        os.environ["VNT_PROFILE_KERNELS"] = "0"
        pe.add_device(work["capacity"])
        pe.set_params(np.concatenate(params))
        mine = node_device >= 0
        with ClockSampler(local) as prof_clocks:   # the clock the GEMM times were taken at
            for i in range(min(args.steps, 10)):
                pe.train_step_ptr(xs[i % nb].data_ptr(), ys[i % nb].data_ptr(), B, sizes,
                                  np.where(mine, 0, -1).astype(np.int32), lr, resident=True)
                t = pe.timings()
                gemm_ms += t["gemm_ms"] * args.steps / min(args.steps, 10)
                gemm_fl += t["gemm_flops"] * args.steps / min(args.steps, 10)
                gemm_n += t["gemm_launches"] * args.steps / min(args.steps, 10)
        line["roofline_clocks"] = prof_clocks.summary()
        line["passes_per_step"] = int(pe.timings()["passes"])
        pe.close()
        line["gpu_launches_note"] = "timed region ran as CUDA-graph replays (one graph per step)"
    if gemm_n and gemm_ms > 0:
        achieved = gemm_fl / (gemm_ms / 1e3) / 1e12
        mode = args.gemm_mode
        if mode in ("auto", "3xtf32"):
            mode = "3xf16"   # VNT_GEMM_AUTO = tcgen05 split-fp16 for wide layers (vnt_engine.h)
        alt = None
        if mode == "ffma":
            peak = 148 * 128 * 2 * (peaks.get("sm_max_mhz", 1965.0) * 1e6) / 1e12
            peak_note = "fp32 FFMA peak 148 SM x 128 FMA/clk x 2 x sm_max_mhz"
        elif mode == "3xf16":
            # kind::f16 runs at the bf16 rate: the driver's measured bf16 dense
            # burst (MEASURED_PEAKS.json) / 3 for the three MMA passes
            # (hi*hi + hi*lo + lo*hi).  Beside it: the sustained figure (the GEMMs
            # run inside a long step), the clock-level ceiling at the median SM
            # clock of the timed region (148 SM x 8192 f16 flop/clk,
            # scripts/ubench_mma_rate.cu) and the nominal 2.25 PF.
            peak = peaks["bf16_tflops"] / 3
            peak_note = f"bf16/f16 dense burst {peaks['bf16_tflops']:.1f} TFLOP/s ({peak_src}) / 3 MMA passes"
            sm_mhz = ((line.get("roofline_clocks") or {}).get("sm_mhz") or (line.get("clocks") or {}).get("sm_mhz")
                      or peaks.get("sm_max_mhz", 1965.0))
            alt = {}
            if peaks.get("bf16_tflops_sustained"):
                sus = peaks["bf16_tflops_sustained"] / 3
                alt["bf16_sustained"] = {"peak": sus, "frac": achieved / sus,
                                         "source": f"bf16 dense sustained ({peak_src}) / 3"}
            ck = 148 * 8192 * sm_mhz * 1e6 / 1e12 / 3
            alt["clock_level"] = {"peak": ck, "frac": achieved / ck,
                                  "source": f"148 SM x 8192 f16 flop/clk x median SM clock {sm_mhz:.0f} MHz"
                                            " while the GEMM launches were timed / 3"}
            alt["nominal"] = {"peak": 2250.0 / 3, "frac": achieved / (2250.0 / 3),
                              "source": "2.25 PFLOP/s dense f16 nominal / 3"}
        else:
            # 1-pass TF32.  MEASURED_PEAKS.json has no TF32 figure: the
            # denominator is the documented fallback, 1.1 PFLOP/s dense TF32
            # (B200_PROFILING.md).  Beside it: the clock-level ceiling at
            # the median SM clock of the timed region (148 SM x 4096 TF32
            # flop/clk, scripts/ubench_mma.cu), cuBLAS TF32 measured here, and
            # the driver's bf16 burst / 2.
            passes = 1
            peak = 1100.0 / passes
            peak_note = ("TF32 dense 1.1 PFLOP/s (fallback, B200_PROFILING.md; no TF32 figure in "
                         "MEASURED_PEAKS.json)")
            tf32_meas = measure_tf32_peak()
            sm_mhz = (line.get("clocks") or {}).get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
            clock_peak = 148 * 4096 * sm_mhz * 1e6 / 1e12 / passes
            derived = peaks["bf16_tflops"] / 2 / passes
        line["roofline"] = {
            "bound": "tensor", "kernel": "dense-layer GEMMs (fwd, bwd-data, per-node dW)",
            "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": None, "peak_source": peak_note,
            "gemm_share_of_step": (gemm_ms / args.steps) / ms_per_step,
            "algorithmic_flops_per_step": flops_step,
            "gemm_launches_per_step": gemm_n / args.steps,
            "alt_peaks": alt if mode != "tf32" else {
                "clock_level": {"peak": clock_peak, "frac": achieved / clock_peak,
                                "source": f"148 SM x 4096 TF32 flop/clk x median SM clock {sm_mhz:.0f} MHz"
                                          " of the timed region" + (", /3" if passes == 3 else "")},
                "cublas_tf32_measured": {"peak": tf32_meas / passes, "frac": achieved / (tf32_meas / passes),
                                         "source": "cuBLAS TF32 8192^3 held 3 s on this GPU"
                                                   + (", /3" if passes == 3 else "")},
                "bf16_burst_half": {"peak": derived, "frac": achieved / derived,
                                    "source": f"bf16 burst / 2 ({peak_src})" + (", /3" if passes == 3 else "")}},
        }
        # DRAM bytes per GEMM launch from the committed `ncu --set full` capture of
        # this workload and mode (profiles/), next to the algorithmic operand bytes.
        prof = ROOT / "profiles" / "r02_ncu_gemm_3xf16.json"
        if prof.exists() and args.workload == "cfg3" and args.gemm_mode in ("auto", "3xf16", "3xtf32"):
            pj = json.loads(prof.read_text())
            line["roofline"]["traffic"] = pj["mean_dram_bytes_per_gemm_launch"]
            line["roofline"]["traffic_unit"] = "bytes/launch (ncu dram__bytes_read+write)"
            line["roofline"]["traffic_source"] = str(prof.relative_to(ROOT))
    eng.close()
    if args.gemm_mode == "auto" and not args.no_extra and "roofline" in line:
        # Secondary: the same step with 1-pass TF32 GEMMs (TF32-grade tolerance,
        # tests/test_tc_gpu.py), timed the same way on the same resident batches.
        fast = vnt.Engine(w, work["act"], work["loss"], cuda_device=local, rank=rank,
                          world_size=world, nccl_id=None if world == 1 else nccl_id,
                          gemm_mode="tf32", resident_rows=args.resident_rows) if world == 1 else None
        if fast is not None:
            fast.add_device(work["capacity"])
            fast.set_params(np.concatenate(params))
            fstream = torch.cuda.ExternalStream(fast.stream_ptr())
            for i in range(args.warmup):
                fast.train_step_ptr(xs[i % nb].data_ptr(), ys[i % nb].data_ptr(), B, sizes,
                                    node_device, lr, resident=True)
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            fms, ffl = 0.0, 0.0
            f0.record(fstream)
            for i in range(args.steps):
                fast.train_step_ptr(xs[i % nb].data_ptr(), ys[i % nb].data_ptr(), B, sizes,
                                    node_device, lr, resident=True)
            f1.record(fstream)
            torch.cuda.synchronize()
            fstep = f0.elapsed_time(f1) / args.steps
            fast.close()
            # GEMM timings from a short eager profiled run, as for the headline line
            os.environ["VNT_PROFILE_KERNELS"] = "1"
            fast = vnt.Engine(w, work["act"], work["loss"], cuda_device=local, gemm_mode="tf32",
                              resident_rows=args.resident_rows)
            os.environ["VNT_PROFILE_KERNELS"] = "0"
            fast.add_device(work["capacity"])
            fast.set_params(np.concatenate(params))
            for i in range(min(args.steps, 8)):
                fast.train_step_ptr(xs[i % nb].data_ptr(), ys[i % nb].data_ptr(), B, sizes,
                                    node_device, lr, resident=True)
                t = fast.timings()
                fms += t["gemm_ms"]
                ffl += t["gemm_flops"]
            tf32_peak = peaks["bf16_tflops"] / 2
            line["also_tf32_1pass"] = {
                "value": B / (fstep / 1e3), "unit": "samples/s", "ms_per_step": fstep,
                "gemm_tflops": ffl / (fms / 1e3) / 1e12 if fms else None,
                "roofline_frac": (ffl / (fms / 1e3) / 1e12) / tf32_peak if fms else None,
                "peak_tflops": tf32_peak,
                "note": "gemm_mode tf32: 1 tcgen05 pass, TF32-grade parity (DESIGN.md §3)"}
            fast.close()
    if "roofline" not in line:
        # Latency-bound small model (whole-node kernel path, no GEMM launches):
        # algorithmic HBM bytes of the step over the step time, against the copy peak.
        P = sum(w[i] * w[i + 1] + w[i + 1] for i in range(len(w) - 1))
        step_bytes = B * (w[0] + w[-1]) * 8 + P * (8 + 8 + 8 + 4 + 4)
        achieved = step_bytes / (ms_per_step / 1e3) / 1e9
        line["roofline"] = {
            "bound": "hbm", "kernel": "whole step (k_node_step + SGD), latency-bound",
            "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"], "traffic": None,
            "algorithmic_bytes_per_step": step_bytes,
            "note": "SURVEY 8(d): cfg1/2 are launch/latency bound; the fraction is reported, "
                    "not optimised against"}
    if rank == 0 and world == 1 and not args.no_extra and args.workload == "cfg3":
        # BASELINE configs[1] (the reference's smallest MLP, V=16) measured by the same
        # script in a child process, reported beside the GEMM-bound headline.
        cmd = [sys.executable, str(ROOT / "bench.py"), "--workload", "cfg1", "--no-extra",
               "--no-cpu-baseline", "--steps", str(max(20 * args.steps, 300)),
               "--warmup", str(max(args.warmup, 10))]
        try:
            out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
            sub = json.loads(out.stdout.strip().splitlines()[-1])
            line["also_cfg2"] = {k: sub[k] for k in ("value", "unit", "ms_per_step", "e2e",
                                                      "config", "gpu_launches", "roofline")}
        except Exception as ex:   # the headline line must still print
            line["also_cfg2"] = {"error": str(ex)[:200]}
    if rank == 0 and world == 1 and not args.no_extra and args.workload == "cfg3":
        # BASELINE configs[3] (cfg4: B = 65536, V = 256 nodes of 256 rows, memory
        # capacity 256 per node): pass rows from free HBM (one pass), and a
        # constrained budget of 4096 resident rows (16 passes) that must give the
        # same bits.
        sub4 = {}
        for tag, rr in (("hbm_sized", 0), ("resident_4096", 4096)):
            cmd = [sys.executable, str(ROOT / "bench.py"), "--workload", "cfg4", "--no-extra",
                   "--no-cpu-baseline", "--steps", "3", "--warmup", "1", "--resident-rows", str(rr)]
            try:
                out = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
                sub = json.loads(out.stdout.strip().splitlines()[-1])
                sub4[tag] = {k: sub.get(k) for k in ("value", "unit", "ms_per_step", "passes_per_step",
                                                     "final_loss", "e2e")}
            except Exception as ex:
                sub4[tag] = {"error": str(ex)[:200]}
        if all("final_loss" in v for v in sub4.values()):
            sub4["same_bits"] = sub4["hbm_sized"]["final_loss"] == sub4["resident_4096"]["final_loss"]
        sub4["config"] = {"workload": "cfg4", "baseline_config_index": 3, "global_batch": 65536,
                          "virtual_nodes": 256, "memory_capacity": 256}
        line["also_cfg4"] = sub4
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base, _ = cpu_reference(work, 1, 0)
        line["cpu_baseline"] = base
        if work["widths"][1] > 256:
            try:
                line["parity"] = headline_parity(vnt, work)
            except Exception as ex:
                line["parity"] = {"error": str(ex)[:200]}
    if world > 1:
        # the reduction the sharded step issues per layer, alone: int64
        # reduce-scatter of the gradient buffer, over this node's NVLink
        P = sum(w[i] * w[i + 1] + w[i + 1] for i in range(len(w) - 1))
        t = torch.ones(((P + world - 1) // world) * world, dtype=torch.int64, device="cuda")
        o = torch.empty(t.numel() // world, dtype=torch.int64, device="cuda")
        for _ in range(2):
            dist.reduce_scatter_tensor(o, t)
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(5):
            dist.reduce_scatter_tensor(o, t)
        c1.record()
        torch.cuda.synchronize()
        rs_ms = c0.elapsed_time(c1) / 5
        line["nccl_int64_reduce_scatter"] = {
            "bytes": t.numel() * 8, "ms": rs_ms,
            "busbw_gbs": t.numel() * 8 * (world - 1) / world / (rs_ms / 1e3) / 1e9}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gemm-mode", default="auto", choices=["auto", "ffma", "tf32", "3xf16", "3xtf32"])
    ap.add_argument("--resident-rows", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true",
                    help="time eager launches with CUDA events around every GEMM (no graphs)")
    ap.add_argument("--no-prefetch", action="store_true",
                    help="e2e: stage each batch inside its own step instead of prefetching")
    ap.add_argument("--no-extra", action="store_true", help="skip the secondary 1-pass TF32 timing")
    args = ap.parse_args()
    work = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, work)
    else:
        run_ours(args, work)


if __name__ == "__main__":
    main()
