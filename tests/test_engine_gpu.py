"""Parity of the B200 engine (through the C-ABI) against the CPU oracle.

Tolerances: FFMA fp32 path — per-step loss within 2e-5
relative and final weights within 2e-5 absolute of the fp64 reference over
the stated steps; TF32 paths are tested in test_tc_gpu.py.  Mapping
invariance (bit-identity for any device count / mapping / pass grouping) is
exact, by construction of the int64 gradient sum.
"""
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


def vnt():
    import paper_2009_09523_b200 as m
    return m


def make_engine(widths, act, loss, seed, port, n_devices=1, capacity=1 << 30, **kw):
    e = vnt().Engine(widths, act, loss, **kw)
    for _ in range(n_devices):
        e.add_device(capacity)
    e.set_params(port.init_params(widths, seed))
    return e


def run(port, widths, act, loss, seed, B, V, lr, ds, n, G, steps, mapping=None, **kw):
    e = make_engine(widths, act, loss, seed, port, n_devices=G, **kw)
    sizes, dev = mapping if mapping is not None else vnt().uniform_mapping(B, V, G)
    losses, metrics = [], None
    for s in range(steps):
        x, y = port.synth_batch(ds, n, widths[0], widths[-1], (s * B) % n, B)
        lo, metrics = e.train_step(x, y, sizes, dev, lr)
        losses.append(lo)
    return e, np.array(losses), metrics


def golden(name):
    z = np.load(GOLDEN / f"ref_{name}.npz")
    return z, json.loads(str(z["config"]))


@pytest.mark.parametrize("name,steps", [("headline", 200), ("cfg1", 20), ("wide_small", 4)])
def test_trajectory_matches_reference(port, name, steps):
    z, c = golden(name)
    e, losses, _ = run(port, c["widths"], c["act"], c["loss"], c["seed"], c["B"], c["V"], c["lr"],
                       c["data_seed"], c["dataset_size"], c["devices"], steps, gemm_mode="ffma")
    rel = np.abs(losses - z["losses"][:steps]) / np.abs(z["losses"][:steps])
    dw = np.abs(e.get_params() - z["params"]).max()
    print(f"{name}: max rel loss dev {rel.max():.3e}, max |dw| {dw:.3e}")
    assert rel.max() <= 2e-5
    assert dw <= 2e-5


def test_input_stats_bit_identical_to_reference(port):
    """LayerStats (model.cpp:101-139) are fp64 in the reference's op order."""
    z, c = golden("cfg1")
    e, _, _ = run(port, c["widths"], c["act"], c["loss"], c["seed"], c["B"], c["V"], c["lr"],
                  c["data_seed"], c["dataset_size"], 1, c["steps"], gemm_mode="ffma")
    cnt, mean, m2 = e.input_stats(0)
    assert cnt == float(z["stats_count"])
    assert np.array_equal(mean, z["stats_mean"])
    assert np.array_equal(m2, z["stats_m2"])


@pytest.mark.parametrize("gemm_mode", ["ffma", "auto"])
def test_bitwise_identical_across_device_counts(port, gemm_mode):
    """test_virtual_exec.cpp:164-182 / acceptance criterion 1, on the GPU path:
    1/2/4/8 devices (and 3, 6 — any mapping) give bit-identical trajectories."""
    w = [64, 96, 48, 10]
    finals, traj = [], []
    for G in (1, 2, 4, 8, 3, 6):
        e, losses, m = run(port, w, "relu", "softmax-cross-entropy", 23, 96, 24, 0.05, 8, 96 * 8,
                           G, 6, gemm_mode=gemm_mode)
        finals.append(e.get_params())
        traj.append(losses)
        assert sum(d["waves"] for d in m) == 24
    for f, t in zip(finals[1:], traj[1:]):
        assert np.array_equal(f, finals[0])
        assert np.array_equal(t, traj[0])


def test_bitwise_identical_across_pass_grouping(port):
    """Resident-row budgets (how many nodes share a pass) never change bits."""
    w = [32, 64, 64, 4]
    outs = []
    for rr in (0, 8, 16, 40):
        e, losses, _ = run(port, w, "tanh", "mse", 3, 64, 8, 0.05, 4, 256, 2, 4,
                           gemm_mode="ffma", resident_rows=rr)
        outs.append((e.get_params(), losses))
    for p, l in outs[1:]:
        assert np.array_equal(p, outs[0][0]) and np.array_equal(l, outs[0][1])


def test_uneven_mapping_matches_even_within_tolerance(port):
    """test_virtual_exec.cpp:218-240: node sizes 6:2 vs 4:4 (different partition,
    so only tolerance-equal), and the 6:2 split on 2 devices == on 1 device bitwise."""
    w = [3, 6, 2]
    x, y = port.synth_batch(11, 8, 3, 2, 0, 8)
    res = []
    for sizes, dev, G in (([6, 2], [0, 1], 2), ([6, 2], [0, 0], 1), ([4, 4], [0, 1], 2)):
        e = make_engine(w, "tanh", "mse", 37, port, n_devices=G, gemm_mode="ffma")
        e.train_step(x, y, sizes, dev, 0.05)
        res.append(e.get_params())
    assert np.array_equal(res[0], res[1])
    assert np.abs(res[0] - res[2]).max() <= 1e-6


def test_device_step_sync_sgd_decomposition(port):
    """device_step / sync_gradients / sgd_apply (virtual_exec.cpp:120-168,
    model.cpp:364-374) through the C-ABI: the synced mean gradient matches the
    full-batch oracle (test_virtual_exec.cpp:115-131, 6:2 weighted sync) and the
    decomposed step equals the fused train_step bit-for-bit."""
    w = [3, 6, 2]
    p0 = port.init_params(w, 13)
    x, y = port.synth_batch(5, 8, 3, 2, 0, 8)
    want, want_loss = port.forward_backward(w, "tanh", "mse", p0, x, y)
    e = make_engine(w, "tanh", "mse", 13, port, n_devices=2, gemm_mode="ffma")
    m0 = e.device_step(0, x[:6], y[:6], [6])
    m1 = e.device_step(1, x[6:], y[6:], [2])
    assert (m0["waves"], m0["examples"], m1["examples"]) == (1, 6, 2)
    g, loss_sum, ex = e.sync()
    assert ex == 8
    assert np.abs(g - want).max() <= 1e-6 * max(1.0, np.abs(want).max())
    assert abs(loss_sum / 8 - want_loss) <= 1e-6
    e.sgd_apply(0.05)
    f = make_engine(w, "tanh", "mse", 13, port, n_devices=2, gemm_mode="ffma")
    f.train_step(x, y, [6, 2], [0, 1], 0.05)
    assert np.array_equal(e.get_params(), f.get_params())


def test_buffer_bytes_and_waves(port):
    """acceptance criterion 10: buffer_bytes == 8*|params| for every V; waves == V."""
    w = [4, 16, 4]
    P = vnt().param_count(w)
    x, y = port.synth_batch(11, 64, 4, 4, 0, 32)
    for V in (1, 2, 4, 8, 16):
        e = make_engine(w, "tanh", "mse", 43, port, n_devices=1, capacity=2048, gemm_mode="ffma")
        sizes, dev = vnt().uniform_mapping(32, V, 1)
        _, m = e.train_step(x, y, sizes, dev, 0.05)
        assert m[0] == {"waves": V, "examples": 32, "peak_resident": 32 // V, "buffer_bytes": 8 * P}


def test_momentum_matches_cpu_restatement(port):
    """Momentum has no reference oracle (model.cpp:364-374 is plain SGD); check
    against our CPU restatement v <- mu v + g; w <- w - lr v on oracle grads."""
    w = [8, 16, 3]
    mu, lr = 0.9, 0.05
    e = make_engine(w, "tanh", "softmax-cross-entropy", 5, port, gemm_mode="ffma", momentum=mu)
    p = port.init_params(w, 5)
    v = np.zeros_like(p)
    sizes, dev = vnt().uniform_mapping(32, 4, 1)
    for s in range(5):
        x, y = port.synth_batch(2, 128, 8, 3, s * 32, 32)
        e.train_step(x, y, sizes, dev, lr)
        g, _ = port.forward_backward(w, "tanh", "softmax-cross-entropy", p, x, y)
        v = mu * v + g
        p = p - lr * v
    assert np.abs(e.get_params() - p).max() <= 1e-5


def test_rescale_retry_keeps_trajectory(port):
    """Force a fixed-point overflow: the engine lowers the scale, redoes the step
    (input statistics observed once) and stays on the reference trajectory."""
    z, c = golden("headline")
    e = make_engine(c["widths"], c["act"], c["loss"], c["seed"], port, gemm_mode="ffma")
    sizes, dev = vnt().uniform_mapping(c["B"], c["V"], 1)
    x, y = port.synth_batch(c["data_seed"], c["dataset_size"], 4, 4, 0, c["B"])
    e.train_step(x, y, sizes, dev, c["lr"])
    e.set_scales(np.full(e.ntensors, 90, np.int32))
    x, y = port.synth_batch(c["data_seed"], c["dataset_size"], 4, 4, c["B"], c["B"])
    lo, _ = e.train_step(x, y, sizes, dev, c["lr"])
    assert e.timings()["rescale_retries"] >= 1
    assert abs(lo - z["losses"][1]) <= 2e-5 * abs(z["losses"][1])
    cnt, _, _ = e.input_stats(0)
    assert cnt == 2 * c["B"]


def test_errors_mirror_reference_exceptions(port):
    V = vnt()
    e = make_engine([3, 6, 2], "tanh", "mse", 1, port, n_devices=1, capacity=4)
    x, y = port.synth_batch(1, 16, 3, 2, 0, 16)
    with pytest.raises(V.VntError) as ei:      # CapacityError
        e.train_step(x, y, [8, 8], [0, 0], 0.05)
    assert ei.value.code == 3
    with pytest.raises(V.VntError) as ei:      # ConfigError: sizes != batch
        e.train_step(x, y, [4, 4], [0, 0], 0.05)
    assert ei.value.code == 2
    with pytest.raises(V.VntError) as ei:      # ConfigError: lr <= 0
        e.train_step(x, y, [4] * 4, [0] * 4, 0.0)
    assert ei.value.code == 2
    with pytest.raises(V.VntError) as ei:      # ShapeError
        e.set_params(np.zeros(3))
    assert ei.value.code == 6
    with pytest.raises(V.VntError) as ei:      # empty node list
        e.device_step(0, x[:0], y[:0], [])
    assert ei.value.code == 2


def test_regroup_single_process_keeps_state(port):
    """vnt_engine_regroup to a 1-process group keeps params, scales and the trajectory."""
    w = [8, 16, 3]
    a = make_engine(w, "tanh", "softmax-cross-entropy", 5, port, gemm_mode="ffma")
    b = make_engine(w, "tanh", "softmax-cross-entropy", 5, port, gemm_mode="ffma")
    sizes, dev = vnt().uniform_mapping(32, 4, 1)
    for s in range(4):
        x, y = port.synth_batch(2, 128, 8, 3, s * 32, 32)
        if s == 2:
            b.regroup(0, 1, None, 0)
        la, _ = a.train_step(x, y, sizes, dev, 0.05)
        lb, _ = b.train_step(x, y, sizes, dev, 0.05)
        assert la == lb
    assert np.array_equal(a.get_params(), b.get_params())
    assert np.array_equal(a.scales(), b.scales())


@pytest.mark.parametrize("graphs,mode", [(True, "auto"), (False, "auto"), (True, "ffma")])
def test_prefetch_is_bit_identical(port, monkeypatch, graphs, mode):
    """vnt_engine_prefetch (runner.cpp:64-73 on the device): staging batch i+1 on
    the copy stream while step i runs — hits, a queued request, a stale
    prefetch (different pointers) — never changes bits."""
    import torch
    if not graphs:
        monkeypatch.setenv("VNT_GRAPHS", "0")
    w = [64, 96, 48, 10]
    steps, B = 7, 96
    xs, ys = [], []
    for s in range(steps):
        x, y = port.synth_batch(8, 96 * 8, 64, 10, (s * B) % (96 * 8), B)
        xs.append(torch.from_numpy(x).pin_memory())
        ys.append(torch.from_numpy(y).pin_memory())
    sizes, dev = vnt().uniform_mapping(B, 24, 1)
    a = make_engine(w, "relu", "softmax-cross-entropy", 23, port, gemm_mode=mode)
    b = make_engine(w, "relu", "softmax-cross-entropy", 23, port, gemm_mode=mode)
    la, lb = [], []
    for s in range(steps):
        la.append(a.train_step_ptr(xs[s].data_ptr(), ys[s].data_ptr(), B, sizes, dev, 0.05, False))
    ptr = lambda i: (xs[i].data_ptr(), ys[i].data_ptr())
    b.prefetch_ptr(*ptr(0), B, sizes, dev, resident=False)
    for s in range(steps):
        if s == 3:
            # stale: the queued batch is 5, step 4 discards it and stages itself
            b.prefetch_ptr(*ptr(5), B, sizes, dev, resident=False)
        elif s + 1 < steps:
            b.prefetch_ptr(*ptr(s + 1), B, sizes, dev, resident=False)
        lb.append(b.train_step_ptr(*ptr(s), B, sizes, dev, 0.05, False))
    assert la == lb
    assert np.array_equal(a.get_params(), b.get_params())


@pytest.mark.parametrize("overlap,shard,w,mode", [("1", "1", [128, 256, 256, 10], "auto"),
                                                  ("0", "1", [128, 256, 256, 10], "auto"),
                                                  ("1", "0", [128, 256, 256, 10], "auto"),
                                                  ("0", "0", [128, 256, 256, 10], "auto"),
                                                  ("1", "1", [64, 96, 48, 10], "ffma")])
def test_collective_paths_bit_identical(port, monkeypatch, overlap, shard, w, mode):
    """VNT_FORCE_COMM=1 gives the engine a one-rank NCCL group, so the collective
    code runs on one GPU: the sharded update (reduce-scatter, 1/G update,
    deferred weight all-gather; default) or the all-reduce + full update
    (VNT_SHARD=0), each in line (VNT_COMM_OVERLAP=0) or overlapped with the
    backward / next forward on a comm stream and captured in the step graph,
    must leave every bit of the trajectory unchanged, for any pass grouping."""
    sizes, dev = vnt().uniform_mapping(256, 8, 1)

    def trajectory(rr):
        e = make_engine(w, "relu", "softmax-cross-entropy", 4, port, gemm_mode=mode,
                        resident_rows=rr)
        losses = []
        for s in range(5):   # steps 2.. replay the captured graph
            x, y = port.synth_batch(4, 2048, w[0], w[-1], s * 256, 256)
            losses.append(e.train_step(x, y, sizes, dev, 0.02)[0])
        return e.get_params(), losses

    want = trajectory(0)
    monkeypatch.setenv("VNT_FORCE_COMM", "1")
    monkeypatch.setenv("VNT_COMM_OVERLAP", overlap)
    monkeypatch.setenv("VNT_SHARD", shard)
    for rr in (0, 96):
        got = trajectory(rr)
        assert got[1] == want[1]
        assert np.array_equal(got[0], want[0])


@pytest.mark.parametrize("widths", [[784, 16, 10], [128, 256, 256, 10]])
def test_resident_batches_match_host_batches(port, widths):
    """Device-resident batches are staged inside the captured step graph
    (k_stage_rows, pointers via the step parameters), host batches by copies:
    rotating resident batches through one graph give the host-path bits."""
    import torch
    B = 128
    sizes, dev = vnt().uniform_mapping(B, 8, 1)
    batches = [port.synth_batch(6, 4096, widths[0], widths[-1], s * B, B) for s in range(3)]
    res = []
    for resident in (False, True):
        e = make_engine(widths, "relu", "softmax-cross-entropy", 9, port, gemm_mode="auto")
        dx = [torch.from_numpy(x).cuda() for x, _ in batches]
        dy = [torch.from_numpy(y).cuda() for _, y in batches]
        losses = []
        for s in range(7):   # graph captured on the 2nd step, replayed with new pointers
            x, y = batches[s % 3]
            if resident:
                losses.append(e.train_step_ptr(dx[s % 3].data_ptr(), dy[s % 3].data_ptr(), B,
                                               sizes, dev, 0.02, resident=True))
            else:
                losses.append(e.train_step(x, y, sizes, dev, 0.02)[0])
        res.append((e.get_params(), losses))
    assert res[0][1] == res[1][1]
    assert np.array_equal(res[0][0], res[1][0])


@pytest.mark.parametrize("widths,mode", [([64, 96, 48, 10], "ffma"), ([64, 96, 48, 10], "auto"),
                                         ([128, 256, 256, 10], "auto")])
def test_rank_partition_sums_add_up_exactly(port, widths, mode):
    """The N > 1 contract on one GPU: processes holding disjoint node sets
    (round-robin, as make_uniform_mapping deals them to ranks) produce exact
    local sums that add up to the single-process sum bit for bit — what the
    int64 NCCL all-reduce then does across GPUs (whole-node kernel, layered
    FFMA + tcgen05, all-tcgen05)."""
    V, m = 8, 16
    B = V * m
    x, y = port.synth_batch(8, 4096, widths[0], widths[-1], 0, B)
    p0 = port.init_params(widths, 3)
    nt = 2 * (len(widths) - 1)

    def local_sum(nodes):
        e = vnt().Engine(widths, "relu", "softmax-cross-entropy", gemm_mode=mode)
        e.add_device(1 << 20)
        e.set_params(p0)
        e.set_scales(np.full(nt, 30, np.int32))   # every process quantises at the same scale
        rows = np.concatenate([np.arange(n * m, (n + 1) * m) for n in nodes])
        e.device_step(0, x[rows], y[rows], [m] * len(nodes))
        g, loss, ex = e.take_gradient_sum()
        e.close()
        return g, loss, ex

    g_all, l_all, ex_all = local_sum(list(range(V)))
    for world in (2, 4):
        parts = [local_sum([n for n in range(V) if n % world == r]) for r in range(world)]
        g = np.sum([p[0] for p in parts], axis=0)
        assert np.array_equal(g, g_all)
        assert sum(p[2] for p in parts) == ex_all == B
        assert abs(sum(p[1] for p in parts) - l_all) <= 1e-9 * abs(l_all)


@pytest.mark.parametrize("widths,mode", [([4, 16, 4], "auto"), ([64, 96, 48, 10], "ffma"),
                                         ([128, 256, 256, 10], "auto")])
def test_zero_params_loss_is_mean_square_label(port, widths, mode):
    """test_model.cpp:76-91 on the engine: with all parameters zero the network
    outputs zero, so the MSE loss is mean(y^2) over the output width (every path:
    whole-node kernel, layered FFMA, tcgen05)."""
    e = vnt().Engine(widths, "tanh", "mse", gemm_mode=mode)
    e.add_device(1 << 20)
    e.set_params(np.zeros(vnt().param_count(widths)))
    x, y = port.synth_batch(2, 512, widths[0], widths[-1], 0, 64)
    sizes, dev = vnt().uniform_mapping(64, 8, 1)
    loss, _ = e.train_step(x, y, sizes, dev, 0.01)
    want = float(np.mean(np.sum(y * y, axis=1) / widths[-1]))
    assert abs(loss - want) <= 1e-9 * want


def test_collective_sequence_node_path(port, monkeypatch):
    """Small models (whole-node kernel) reduce G and its tail in one call on
    every rank layout."""
    monkeypatch.setenv("VNT_FORCE_COMM", "1")
    w = [64, 96, 48, 10]
    sizes, _ = vnt().uniform_mapping(128, 8, 1)
    x, y = port.synth_batch(4, 2048, w[0], w[-1], 0, 128)
    logs = []
    for node_device in ([0] * 8, [-1] * 8, [0, -1] * 4):
        # ffma: every layer on FFMA kernels, so the whole-node path (auto would put
        # the 64->96 layer on tcgen05 and take the layered path)
        e = make_engine(w, "relu", "softmax-cross-entropy", 4, port, gemm_mode="ffma")
        e.comm_log()
        e.train_step(x, y, sizes, np.array(node_device, np.int32), 0.02)
        logs.append(e.comm_log())
    assert len(logs[0]) == 1 and logs[0][0][:2] == ("allreduce", 0)
    assert logs[1] == logs[0] and logs[2] == logs[0]


def test_collective_sequence_is_rank_independent(port, monkeypatch):
    """Every rank must issue the same collectives in the same order (NCCL
    matches them by order): a process with all nodes, one with none (it
    reduces zeros), and one whose nodes need three passes all log the same
    sequence — sharded update: per layer L-1..0 reduce-scatter (overlapped with
    the backward), the tail all-reduce, the max all-reduce of the split-fp16
    operand maxima (2L+3 words, the update's range check), the max|g|
    all-reduce; from the second step on, first the weight all-gathers of
    layers 0..L-1."""
    monkeypatch.setenv("VNT_FORCE_COMM", "1")
    w = [128, 256, 256, 10]
    sizes, _ = vnt().uniform_mapping(256, 8, 1)
    x, y = port.synth_batch(4, 2048, w[0], w[-1], 0, 256)
    logs = []
    for node_device, rr in (([0] * 8, 0), ([-1] * 8, 0), ([0] * 8, 96)):
        e = make_engine(w, "relu", "softmax-cross-entropy", 4, port, gemm_mode="auto",
                        resident_rows=rr)
        e.comm_log()   # creation-time traffic, if any
        e.train_step(x, y, sizes, np.array(node_device, np.int32), 0.02)
        first = e.comm_log()
        e.train_step(x, y, sizes, np.array(node_device, np.int32), 0.02)
        logs.append((first, e.comm_log()))
    L = len(w) - 1
    offs, p = [], 0
    for l in range(L):
        n = w[l] * w[l + 1] + w[l + 1]
        offs.append((p, (n + 31) // 32 * 32))   # one rank: chunk = slice rounded to 32
        p += n
    rs = [("reduce_scatter", o, c) for o, c in reversed(offs)]
    first, second = logs[0]
    assert first[:L] == rs
    assert [op for op, _, _ in first[L:]] == ["allreduce", "max", "max"]
    assert first[L + 1][2] == 2 * L + 3
    assert second == [("allgather", o, c) for o, c in offs] + first
    assert logs[1] == logs[0] and logs[2] == logs[0]


@pytest.mark.parametrize("w,mode", [([64, 96, 48, 10], "ffma"), ([128, 256, 256, 10], "auto")])
def test_nonfinite_step_raises_and_leaves_state(port, w, mode):
    """ExactAccumulator rejects non-finite values (exact_sum.cpp:17-19): a NaN in
    the batch fails the step with VNT_ERR_NONFINITE, skips the SGD on the
    device and restores the input statistics; the next finite step proceeds."""
    V = vnt()
    e = make_engine(w, "relu", "softmax-cross-entropy", 6, port, gemm_mode=mode)
    sizes, dev = V.uniform_mapping(64, 4, 1)
    x, y = port.synth_batch(5, 1024, w[0], w[-1], 0, 64)
    e.train_step(x, y, sizes, dev, 0.02)
    p1 = e.get_params()
    cnt1, mean1, m21 = e.input_stats(0)
    bad = x.copy()
    bad[3, 5] = np.nan
    with pytest.raises(V.VntError) as ei:
        e.train_step(bad, y, sizes, dev, 0.02)
    assert ei.value.code == 11
    assert np.array_equal(e.get_params(), p1)
    cnt2, mean2, m22 = e.input_stats(0)
    assert cnt2 == cnt1 and np.array_equal(mean2, mean1) and np.array_equal(m22, m21)
    loss, _ = e.train_step(x, y, sizes, dev, 0.02)
    assert np.isfinite(loss)


def test_single_layer_identity_least_squares_known_answer():
    """test_model.cpp:93-111 on the engine: [2,1] identity/MSE, params
    (0.5, -0.25, 0.1), x = (2, 3), y = 1.5 -> residual r = -1.15, loss r^2,
    gradient (2r*2, 2r*3, 2r); fp32 compute, tolerance 1e-6 relative."""
    e = vnt().Engine([2, 1], "identity", "mse", gemm_mode="ffma")
    e.add_device(1 << 20)
    e.set_params(np.array([0.5, -0.25, 0.1]))
    e.device_step(0, np.array([[2.0, 3.0]]), np.array([[1.5]]), [1])
    g, loss_sum, ex = e.sync()
    r = 2.0 * 0.5 + 3.0 * -0.25 + 0.1 - 1.5
    assert ex == 1
    assert abs(loss_sum - r * r) <= 1e-6 * r * r
    want = np.array([2 * r * 2.0, 2 * r * 3.0, 2 * r])
    assert np.abs(g - want).max() <= 1e-6 * np.abs(want).max()
    e.close()


@pytest.mark.parametrize("mode", ["ffma", "3xf16"])
def test_union_gradient_is_size_weighted_mean_of_parts(port, mode):
    """test_model.cpp:148-163: the gradient of a union is the size-weighted mean
    of the parts' gradients.  On the engine the 5:3 split as two virtual nodes
    is compared with the two parts run alone (1e-12, the reference's bound: the
    int64 node sums add exactly; only the fp64 divisions by 8, 5, 3 round)."""
    w = [64, 96, 80, 3] if mode == "3xf16" else [4, 6, 3]
    p0 = port.init_params(w, 33)
    x, y = port.synth_batch(99, 64, w[0], w[-1], 0, 8)

    def grad(xs, ys, sizes):
        e = vnt().Engine(w, "tanh", "softmax-cross-entropy", gemm_mode=mode)
        e.add_device(1 << 20)
        e.set_params(p0)
        e.device_step(0, xs, ys, sizes)
        g, _, _ = e.sync()
        e.close()
        return g

    g = grad(x, y, [5, 3])
    ga, gb = grad(x[:5], y[:5], [5]), grad(x[5:], y[5:], [3])
    expect = (5.0 * ga + 3.0 * gb) / 8.0
    assert np.all(np.abs(g - expect) <= 1e-12 * np.maximum(1.0, np.abs(expect)))
