"""Pin the CPU oracle before trusting it (CPU only, no GPU).

* The plain-C restatement (oracle/vnt_oracle.c) must reproduce the
  reference's own checked-in fig1 outputs (golden, 1e-15 — the survey measured
  <= 5.55e-17 libm/platform differences) and be bit-identical to the
  reference compiled from its sources (oracle/_ref) wherever that exists.
* Golden trajectories produced by the reference (tests/golden/ref_*.npz, made
  by tests/golden/make_golden.py) must be reproduced bit-for-bit by the port.
"""
import json
from pathlib import Path

import numpy as np
import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"


def _case(name):
    z = np.load(GOLDEN / f"ref_{name}.npz")
    cfg = json.loads(str(z["config"]))
    return z, cfg


def test_fig1_reference_outputs(port):
    g = json.loads((GOLDEN / "fig1_reference.json").read_text())
    c = g["config"]
    t = port.trainer(c["layer_widths"], c["activation"], c["loss"], c["seed"], c["global_batch"],
                     c["virtual_nodes"], c["lr"], c["data_seed"], c["dataset_size"], c["devices"])
    losses = np.array([t.step() for _ in range(c["steps"])])
    np.testing.assert_allclose(losses, g["step_losses"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(t.params(), g["final_params"], rtol=0, atol=1e-15)
    # Layout names/shapes as model.cpp:62-77 lays them out.
    assert [n for n, _ in g["layout"]] == ["layer0/weight", "layer0/bias", "layer1/weight", "layer1/bias"]


@pytest.mark.parametrize("name", ["headline", "cfg1"])
def test_port_reproduces_reference_goldens_bitwise(port, name):
    z, c = _case(name)
    steps = min(c["steps"], 20)
    t = port.trainer(c["widths"], c["act"], c["loss"], c["seed"], c["B"], c["V"], c["lr"],
                     c["data_seed"], c["dataset_size"], c["devices"])
    losses = np.array([t.step() for _ in range(steps)])
    assert np.array_equal(losses, z["losses"][:steps])
    if steps == c["steps"]:
        assert np.array_equal(t.params(), z["params"])
        cnt, mean, m2 = t.input_stats(0)
        assert cnt == float(z["stats_count"])
        assert np.array_equal(mean, z["stats_mean"]) and np.array_equal(m2, z["stats_m2"])


def test_port_matches_compiled_reference(port, ref):
    if ref is None:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    w = [3, 6, 2]
    for act in ["relu", "tanh", "identity"]:
        for loss in ["mse", "softmax-cross-entropy"]:
            p = ref.init_params(w, 5)
            assert np.array_equal(p, port.init_params(w, 5))
            x, y = ref.synth_batch(3, 40, 3, 2, 7, 9)
            x2, y2 = port.synth_batch(3, 40, 3, 2, 7, 9)
            assert np.array_equal(x, x2) and np.array_equal(y, y2)
            g1, l1 = ref.forward_backward(w, act, loss, p, x, y)
            g2, l2 = port.forward_backward(w, act, loss, p, x, y)
            assert np.array_equal(g1, g2) and l1 == l2
    # Trainer + resize 8 -> 4 -> 2 -> 6 (elastic.cpp:106-245), stats bitwise.
    a = ref.trainer([4, 16, 4], "tanh", "mse", 11, 64, 8, 0.05, 11, 256, 8)
    b = port.trainer([4, 16, 4], "tanh", "mse", 11, 64, 8, 0.05, 11, 256, 8)
    for s in range(12):
        if s in (3, 6, 9):
            n = {3: 4, 6: 2, 9: 6}[s]
            a.resize(n)
            b.resize(n)
        assert a.step() == b.step()
    assert np.array_equal(a.params(), b.params())
    for i in range(6):
        for u, v in zip(a.input_stats(i), b.input_stats(i)):
            assert np.array_equal(u, v)


def test_mapping_invariance_in_oracle(port):
    """test_virtual_exec.cpp:164-182: bitwise-identical params across 1/2/4/8 devices."""
    finals = []
    for G in (1, 2, 4, 8):
        t = port.trainer([3, 6, 2], "tanh", "mse", 23, 64, 8, 0.05, 8, 64 * 5, G)
        for _ in range(5):
            t.step()
        finals.append(t.params())
    for f in finals[1:]:
        assert np.array_equal(f, finals[0])


def test_finite_differences(port):
    """acceptance.cpp:207-234: analytic grads within 1e-6 of central differences."""
    for act in ["relu", "tanh", "identity"]:
        for loss in ["mse", "softmax-cross-entropy"]:
            w = [3, 5, 4]
            p = port.init_params(w, 1000)
            x, y = port.synth_batch(0, 6, 3, 4, 0, 6)
            g, _ = port.forward_backward(w, act, loss, p, x, y)
            h = 1e-5
            for i in range(p.size):
                pp, pm = p.copy(), p.copy()
                pp[i] += h
                pm[i] -= h
                fd = (port.forward_backward(w, act, loss, pp, x, y)[1]
                      - port.forward_backward(w, act, loss, pm, x, y)[1]) / (2 * h)
                assert abs(fd - g[i]) <= 1e-6 * max(1.0, abs(g[i]))


@pytest.mark.parametrize("widths,act,loss,B", [([64, 96, 48, 10], "relu", "softmax-cross-entropy", 64),
                                               ([32, 64, 4], "tanh", "mse", 37),
                                               ([784, 256, 10], "relu", "softmax-cross-entropy", 16)])
def test_wide_oracle_pinned_to_exact_oracle(port, widths, act, loss, B):
    """vo_forward_backward_wide (the checker of the headline-width GPU tests)
    against the exactly rounded vo_forward_backward: same per-example
    arithmetic, compensated instead of exact sums — loss bit-identical,
    gradients within 4 ulp of the element's magnitude."""
    p = port.init_params(widths, 5)
    x, y = port.synth_batch(9, 1024, widths[0], widths[-1], 3, B)
    g0, l0 = port.forward_backward(widths, act, loss, p, x, y)
    g1, l1 = port.forward_backward_wide(widths, act, loss, p, x, y)
    assert l1 == l0
    ulp = np.spacing(np.abs(g0)) + np.spacing(np.abs(g0).max()) * 1e-6
    assert np.all(np.abs(g1 - g0) <= 4 * ulp)
