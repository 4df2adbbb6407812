"""The skinny-layer backward variants give the same bits: the bulk-copy
streamed kernel with packed FFMA2 (k_skinny_backward_bulk, default when
in % 4 == 0) against the register-pipelined two-features-per-thread kernel
(k_skinny_backward2, VNT_SKINNY_BULK=0).  The choice is read once per process,
so each variant trains in its own subprocess; ragged node sizes (125 / 131
rows: partial 8-row stages and pad rows) and a 4096-wide last hidden layer
feeding the 10-output skinny layer, as at cfg3."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, %(root)r)
import paper_2009_09523_b200 as vnt
widths = %(widths)r
B = %(B)d
g = torch.Generator(device="cuda").manual_seed(5)
T = torch.randn(widths[0], widths[-1], device="cuda", dtype=torch.float64, generator=g) / 28.0
r = np.random.default_rng(3)
ps = []
for i in range(len(widths) - 1):
    ps.append(r.standard_normal(widths[i] * widths[i + 1]) / np.sqrt(widths[i]))
    ps.append(r.standard_normal(widths[i + 1]) * 0.01)
e = vnt.Engine(widths, %(act)r, "softmax-cross-entropy")
e.add_device(1 << 20)
e.set_params(np.concatenate(ps))
sizes = %(sizes)r
dev = [0] * len(sizes)
losses = []
for s in range(3):
    x = torch.randn(B, widths[0], device="cuda", dtype=torch.float64, generator=g)
    y = torch.softmax(x @ T, dim=1)
    losses.append(e.train_step_ptr(x.data_ptr(), y.data_ptr(), B, sizes, dev, 0.05, resident=True))
p = e.get_params()
e.close()
print(json.dumps({"params": hashlib.sha256(np.ascontiguousarray(p).tobytes()).hexdigest(),
                  "losses": [float(v).hex() for v in losses]}))
"""


def _run(bulk, **kw):
    # VNT_NODE_KERNEL=0: small models take the per-layer kernels (not the
    # whole-node kernel), so the skinny backward runs
    env = dict(os.environ, VNT_SKINNY_BULK=str(bulk), VNT_NODE_KERNEL="0")
    out = subprocess.run([sys.executable, "-c", SCRIPT % dict(root=ROOT, **kw)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("act", ["relu", "tanh"])
def test_bulk_backward_bits_equal_register_kernel(act):
    sizes = [125, 131] * 8
    kw = dict(widths=[784, 4096, 4096, 10], B=sum(sizes), act=act, sizes=sizes)
    a, b = _run(1, **kw), _run(0, **kw)
    assert a == b


def test_bulk_backward_partial_slab():
    # a 300-wide hidden layer: the last 256-feature slab holds 44
    # features (176-B rows), odd node sizes
    sizes = [97, 64, 33, 150]
    kw = dict(widths=[784, 300, 10], B=sum(sizes), act="relu", sizes=sizes)
    assert _run(1, **kw) == _run(0, **kw)


@pytest.mark.parametrize("widths,act", [
    ([784, 10], "relu"),                 # layer 0 skinny: dW only (no bwd-data / db)
    ([784, 256, 4], "identity"),         # NO = 4
    ([784, 512, 8], "tanh"),             # NO = 8
    ([784, 256, 16], "relu"),            # NO = 16
    ([784, 128, 32], "identity"),        # NO = 32
])
def test_bulk_backward_instantiations(widths, act):
    sizes = [40, 88, 19, 61]
    kw = dict(widths=widths, B=sum(sizes), act=act, sizes=sizes)
    assert _run(1, **kw) == _run(0, **kw)
