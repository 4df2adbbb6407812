"""Headline-width parity diagnostics: the engine's mean gradient at the cfg3
widths ([784, 4096 x 4, 10], relu, softmax-CE, B = 64, V = 8) against the
fp64 oracle with relu masks resolved in the fp32 band (as
tests/test_headline_parity_gpu.py), per tensor: max deviation relative to
max |g_ref|, and the loss.  usage: python scripts/diag_headline.py [mode]"""
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
e = vnt.Engine(W, "relu", "softmax-cross-entropy", gemm_mode=mode)
e.add_device(1 << 20)
e.set_params(p0)
e.device_step(0, x, y, np.full(V, B // V, np.uint64))
acts = {l: e.debug_activation(l, B) for l in range(1, len(W) - 1)}
g, ls, ex = e.sync()
g_ref, l_ref, flips, conf = port.forward_backward_wide(W, "relu", "softmax-cross-entropy", p0, x, y,
                                                       act_ext=acts, tau=3e-5, counts=True)
print("mode", mode, "loss", ls / ex, l_ref, "masks resolved", flips, "conflicts", conf)
off, worst = 0, 0.0
for l in range(len(W) - 1):
    n = W[l] * W[l + 1]
    for name, a, b in ((f"W{l}", off, off + n), (f"b{l}", off + n, off + n + W[l + 1])):
        m = np.abs(g_ref[a:b]).max()
        d = float(np.abs(g[a:b] - g_ref[a:b]).max() / m)
        worst = max(worst, d)
        print(f"{name}: max|ref| {m:.3e} dev {d:.3e}")
    off += n + W[l + 1]
print(f"max dev {worst:.3e}")
