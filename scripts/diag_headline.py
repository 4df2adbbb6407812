"""Diagnostics for the headline-width parity: per-tensor deviation of the
engine's mean gradient from the fp64 oracle, and where the worst elements sit
(row = input unit, col = output unit)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import oracle_lib
import paper_2009_09523_b200 as vnt

W = [784, 4096, 4096, 4096, 4096, 10]
mode = sys.argv[1] if len(sys.argv) > 1 else "auto"
B, V = 64, 8
port = oracle_lib.port()
p0 = port.init_params(W, 1)
x, y = port.synth_batch(1, 65536, 784, 10, 0, B)
g_ref, l_ref = port.forward_backward_wide(W, "relu", "softmax-cross-entropy", p0, x, y)
e = vnt.Engine(W, "relu", "softmax-cross-entropy", gemm_mode=mode)
e.add_device(1 << 20)
e.set_params(p0)
e.device_step(0, x, y, np.full(V, B // V, np.uint64))
g, ls, ex = e.sync()
print("mode", mode, "loss", ls / ex, l_ref)
off = 0
for l in range(len(W) - 1):
    n = W[l] * W[l + 1]
    for name, a, b, shape in ((f"W{l}", off, off + n, (W[l], W[l + 1])), (f"b{l}", off + n, off + n + W[l + 1], (1, W[l + 1]))):
        gr, gg = g_ref[a:b], g[a:b]
        m = np.abs(gr).max()
        d = np.abs(gg - gr)
        bad = d > 1e-4 * m
        rows, cols = np.nonzero(bad.reshape(shape))
        print(f"{name}: max|ref| {m:.3e} dev {d.max() / m:.3e} n_bad {bad.sum()} "
              f"distinct cols {len(set(cols.tolist()))} rows {len(set(rows.tolist()))} "
              f"cols {sorted(set(cols.tolist()))[:12]}")
    off += n + W[l + 1]
