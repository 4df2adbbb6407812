"""Barrier-wait probe of the tcgen05 GEMMs (diagnostics; run on a scratch copy).

Rebuilds paper_2009_09523_b200/libvnt_engine.so IN PLACE with -DVNT_TC_PROBE,
runs cfg3 steps and prints, per kernel kind, the fraction of each role's
cycles spent waiting: producer on smem-empty, MMA issuer on TMEM-empty and
on smem-full, epilogue on TMEM-full.  Do not commit the probe build.

usage (GPU box): python scripts/tc_probe.py [steps]
Env VNT_TC_DW_PAIR=1 selects the CTA-pair dW kernel.
"""
import ctypes as C
import subprocess
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
PKG = ROOT / "paper_2009_09523_b200"

from paper_2009_09523_b200 import build as b  # noqa: E402

import os  # noqa: E402
extra = os.environ.get("VNT_EXTRA_DEFS", "").split()   # e.g. "-DVNT_EXP_X" for experiments
subprocess.check_call([b.NVCC, *b.ARCH, "-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-DVNT_TC_PROBE", *extra,
                       "-shared", "-o", str(PKG / "libvnt_engine.so"), str(PKG / "csrc" / "engine.cu"),
                       *b.nccl_flags(), "-lcuda"])

import torch  # noqa: E402

import paper_2009_09523_b200 as vnt  # noqa: E402

WIDE = [784, 4096, 4096, 4096, 4096, 10]
B, V = 8192, 64
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
lib = vnt.load_engine()
probe = lib.vnt_debug_tc_probe
buf = (C.c_ulonglong * 96)()

r = np.random.default_rng(1)
params = np.concatenate([np.concatenate([r.standard_normal(WIDE[i] * WIDE[i + 1]) / np.sqrt(WIDE[i]),
                                         np.zeros(WIDE[i + 1])]) for i in range(len(WIDE) - 1)])
x = torch.randn(B, 784, device="cuda", dtype=torch.float64)
y = torch.softmax(torch.randn(B, 10, device="cuda", dtype=torch.float64), dim=1)
e = vnt.Engine(WIDE, "relu", "softmax-cross-entropy", gemm_mode=sys.argv[2] if len(sys.argv) > 2 else "auto")
e.add_device(1 << 20)
e.set_params(params)
sizes, dev = vnt.uniform_mapping(B, V, 1, 1 << 20)
for s in range(2):
    e.train_step_ptr(x.data_ptr(), y.data_ptr(), B, sizes, dev, 0.01, resident=True)
torch.cuda.synchronize()
probe(buf)
t0 = torch.cuda.Event(enable_timing=True)
t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for s in range(steps):
    e.train_step_ptr(x.data_ptr(), y.data_ptr(), B, sizes, dev, 0.01, resident=True)
t1.record()
torch.cuda.synchronize()
print(f"ms/step (probe build) {t0.elapsed_time(t1) / steps:.3f}")
probe(buf)
a = np.array(buf, dtype=np.float64).reshape(6, 16)
names = ["fwd", "bwd", "dW", "pair fwd", "pair bwd", "pair dW"]
for k in range(6):
    if a[k, 1] == 0:
        continue
    print(f"{names[k]:9s} producer wait {a[k, 0] / a[k, 1]:.3f} | MMA tempty wait {a[k, 2] / a[k, 3]:.3f}"
          f" full wait {a[k, 6] / a[k, 3]:.3f} | epilogue tfull wait {a[k, 4] / max(a[k, 5], 1):.3f}"
          f" | MMA-thread cycles/launch-CTA {a[k, 3]:.3e}")
    if a[k, 9]:
        print(f"{'':9s} final epilogue {a[k, 8] / a[k, 9]:.0f} cyc x {a[k, 9]:.0f}"
              + (f" | promote {a[k, 10] / a[k, 11]:.0f} cyc x {a[k, 11]:.0f}" if a[k, 11] else ""))
    if a[k, 12] + a[k, 13] + a[k, 14] + a[k, 15]:
        n = max(a[k, 9], 1) * 4
        print(f"{'':9s} per 32-col finish: bias/act {a[k, 12] / n:.0f} | mask {a[k, 13] / n:.0f} | store wait "
              f"{a[k, 14] / n:.0f} | convert+stage {a[k, 15] / n:.0f} cyc")
e.close()
