"""Engine edge cases found by review, through the C-ABI.

* whole-node kernel: the per-node CTA cluster is a function of the model only,
  so a node's bits never depend on which nodes share its pass (uneven sizes,
  pass groupings, logical device counts);
* per-row loss range: rows whose quantised loss could overflow the int64 loss
  sum force a redo at a coarser quantum instead of wrapping;
* prefetch: a staged batch is used only when it was staged for the same
  mapping, not merely the same pointers;
* int64 headroom: more virtual nodes than the fixed-point format allows is a
  ConfigError, not a silent overflow.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def vnt():
    import paper_2009_09523_b200 as m
    return m


def engine(port, widths, act, loss, seed, devices=1, **kw):
    e = vnt().Engine(widths, act, loss, **kw)
    for _ in range(devices):
        e.add_device(1 << 30)
    e.set_params(port.init_params(widths, seed))
    return e


def test_node_kernel_bits_independent_of_pass_company(port):
    """[784,16,10] (the whole-node path) with one 200-row node among 16-row
    nodes: alone in a pass, sharing a pass, on 1 or 2 logical devices."""
    w = [784, 16, 10]
    sizes = [16] * 8 + [200] + [16] * 4
    B = sum(sizes)
    x, y = port.synth_batch(5, 4096, 784, 10, 0, B)
    runs = []
    for devices, rr in ((1, 0), (1, 128), (2, 0), (2, 216), (1, 200)):
        e = engine(port, w, "tanh", "softmax-cross-entropy", 7, devices=devices, resident_rows=rr)
        dev = [k % devices for k in range(len(sizes))]
        losses = [e.train_step(x, y, sizes, dev, 0.05)[0] for _ in range(3)]
        runs.append((losses, e.get_params()))
        e.close()
    for losses, p in runs[1:]:
        assert losses == runs[0][0]
        assert np.array_equal(p, runs[0][1])


@pytest.mark.parametrize("widths,mode", [([4, 16, 4], "auto"), ([64, 96, 48, 10], "ffma")])
def test_loss_range_redo_keeps_exact_loss(port, widths, mode):
    """MSE against labels of 1e6: row losses ~1e12 overflow 2^62/B at the
    default 2^-32 quantum; the step is redone at a coarser one and the loss
    still equals the fp64 reference to its quantum."""
    B, V = 64, 8
    x, y = port.synth_batch(3, 1024, widths[0], widths[-1], 0, B)
    y = y * 1e6
    e = engine(port, widths, "tanh", "mse", 5, gemm_mode=mode)
    p0 = port.init_params(widths, 5)
    sizes, dev = vnt().uniform_mapping(B, V, 1)
    loss, _ = e.train_step(x, y, sizes, dev, 1e-12)
    assert e.timings()["rescale_retries"] >= 1
    _, want = port.forward_backward(widths, "tanh", "mse", p0, x, y)
    assert abs(loss - want) <= 1e-6 * abs(want), (loss, want)
    # and the quantum comes back once losses are small again
    y2 = y / 1e6
    e.train_step(x, y2, sizes, dev, 1e-12)
    p1 = e.get_params()
    loss2, _ = e.train_step(x, y2, sizes, dev, 1e-12)
    _, want2 = port.forward_backward(widths, "tanh", "mse", p1, x, y2)
    assert abs(loss2 - want2) <= 2e-5 * abs(want2) + 1e-9


def test_prefetch_for_another_mapping_is_not_used(port):
    import torch
    w = [64, 96, 48, 10]
    B = 96
    x, y = port.synth_batch(8, 768, 64, 10, 0, B)
    xt, yt = torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory()
    a = engine(port, w, "relu", "softmax-cross-entropy", 23, devices=2)
    b = engine(port, w, "relu", "softmax-cross-entropy", 23, devices=2)
    s1, d1 = vnt().uniform_mapping(B, 8, 2)
    s2, d2 = [8] * 4 + [16] * 4, [1, 0, 1, 0, 1, 0, 1, 0]
    la = a.train_step_ptr(xt.data_ptr(), yt.data_ptr(), B, s2, d2, 0.05, False)
    b.prefetch_ptr(xt.data_ptr(), yt.data_ptr(), B, s1, d1, resident=False)
    lb = b.train_step_ptr(xt.data_ptr(), yt.data_ptr(), B, s2, d2, 0.05, False)
    assert la == lb
    assert np.array_equal(a.get_params(), b.get_params())


def test_too_many_virtual_nodes_is_a_config_error(port):
    w = [4, 16, 4]
    e = engine(port, w, "tanh", "mse", 1)
    V = (1 << 21) + 1
    x, y = port.synth_batch(1, V, 4, 4, 0, V)
    with pytest.raises(vnt().VntError) as ei:
        e.train_step(x, y, [1] * V, [0] * V, 0.01)
    assert ei.value.kind == "ConfigError"
