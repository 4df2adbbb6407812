"""Host logic of the N > 1 path on CPU with gloo (world_size 2): virtual nodes
dealt round-robin to ranks, each rank quantising its nodes' fp32 gradient
partials to int64 fixed point exactly as the engine's dW epilogue does
(DESIGN.md §3), one integer all-reduce — the reduced sum must be bit-identical
to the single-process sum for every world size and node grouping."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def node_partials(V, m, shape, seed=0):
    """Deterministic fp32 per-node partials (stand-in for g_k = X_k^T D_k)."""
    g = np.random.default_rng(seed)
    out = []
    for k in range(V):
        x = g.standard_normal((m, shape[0])).astype(np.float32)
        d = g.standard_normal((m, shape[1])).astype(np.float32) * np.float32(1e-2)
        out.append((x.T @ d).astype(np.float32))
    return out


def quantise(gk, s):
    v = gk.astype(np.float32) * np.float32(2.0 ** s)
    assert np.all(np.abs(v) < 2.0 ** 50)
    return np.rint(v).astype(np.int64)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, V, m, s, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2009_09523_b200 as vnt
    sizes, dev = vnt.uniform_mapping(V * m, V, world)
    parts = node_partials(V, m, (24, 10))
    local = np.zeros((24, 10), np.int64)
    for k in np.nonzero(dev == rank)[0][::-1]:        # any local order
        local += quantise(parts[k], s)
    t = torch.from_numpy(local)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    q.put((rank, t.numpy().copy(), int((dev == rank).sum())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_int64_allreduce_matches_single_process_bitwise(world):
    V, m, s = 12, 16, 30
    parts = node_partials(V, m, (24, 10))
    want = np.zeros((24, 10), np.int64)
    for k in range(V):
        want += quantise(parts[k], s)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, V, m, s, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert sum(n for _, _, n in got) == V
    for _, arr, _ in got:
        assert np.array_equal(arr, want)
    # the fp32 tree the survey feared: a float sum in another order is NOT invariant
    f1 = np.zeros((24, 10), np.float32)
    f2 = np.zeros((24, 10), np.float32)
    for k in range(V):
        f1 += parts[k]
    for k in reversed(range(V)):
        f2 += parts[k]
    assert not np.array_equal(f1, f2) or world == 1


def _hostcomm_worker(rank, world, port, q):
    """Every callback of the engine's host-callback group (vnt_comm_ops,
    hostcomm.py) exercised through its C function pointers, as the engine's
    HostGroup calls them, on CPU with gloo."""
    import ctypes as C
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2009_09523_b200 import hostcomm
    g = hostcomm.world_group()
    ops, ctx = g.ops, g.ops.ctx
    res = {}
    # int64 sum all-reduce
    a = np.arange(6, dtype=np.int64) + 100 * rank
    assert ops.allreduce(ctx, a.ctypes.data, a.size, 0) == 0
    res["sum"] = a.copy()
    # uint64 max (positive doubles' bit patterns)
    m = np.array([float(rank + 1), 0.5 * rank]).view(np.int64).copy()
    assert ops.allreduce(ctx, m.ctypes.data, m.size, 1) == 0
    res["max"] = m.view(np.float64).copy()
    # reduce-scatter: rank r gets its block of the sum
    send = np.arange(4 * world, dtype=np.int64) * (rank + 1)
    recv = np.zeros(4, np.int64)
    assert ops.reduce_scatter(ctx, send.ctypes.data, recv.ctypes.data, 4) == 0
    res["rs"] = recv.copy()
    # all-gather of bytes
    chunk = np.full(3, rank + 7, np.float32)
    out = np.zeros(3 * world, np.float32)
    assert ops.allgather(ctx, chunk.ctypes.data, out.ctypes.data, chunk.nbytes) == 0
    res["ag"] = out.copy()
    # broadcast from the last rank
    b = np.full(2, rank, np.float64)
    assert ops.broadcast(ctx, b.ctypes.data, b.nbytes, world - 1) == 0
    res["bc"] = b.copy()
    # send/recv ring
    token = np.array([rank * 10.0])
    got = np.zeros(1)
    if rank % 2 == 0:
        assert ops.send(ctx, token.ctypes.data, token.nbytes, (rank + 1) % world) == 0
        assert ops.recv(ctx, got.ctypes.data, got.nbytes, (rank - 1) % world) == 0
    else:
        assert ops.recv(ctx, got.ctypes.data, got.nbytes, (rank - 1) % world) == 0
        assert ops.send(ctx, token.ctypes.data, token.nbytes, (rank + 1) % world) == 0
    res["ring"] = got.copy()
    # split: the even ranks form a group; sum inside it
    sub = hostcomm.CommOps()
    assert ops.split(ctx, 0 if rank % 2 == 0 else -1, rank, C.byref(sub)) == 0
    if rank % 2 == 0:
        s = np.array([rank + 1], np.int64)
        assert sub.allreduce(sub.ctx, s.ctypes.data, 1, 0) == 0
        res["split"] = (int(sub.rank), int(sub.size), int(s[0]))
    else:
        res["split"] = bool(sub.ctx)
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_callback_group_collectives(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hostcomm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    evens = [r for r in range(world) if r % 2 == 0]
    for r, res in out.items():
        assert np.array_equal(res["sum"], world * np.arange(6) + 100 * sum(range(world)))
        assert np.array_equal(res["max"], [float(world), 0.5 * (world - 1)])
        full = sum(np.arange(4 * world) * (k + 1) for k in range(world))
        assert np.array_equal(res["rs"], full[4 * r:4 * r + 4])
        assert np.array_equal(res["ag"], np.repeat(np.arange(world) + 7, 3).astype(np.float32))
        assert np.array_equal(res["bc"], [world - 1] * 2)
        assert res["ring"][0] == ((r - 1) % world) * 10.0
        if r % 2 == 0:
            assert res["split"] == (evens.index(r), len(evens), sum(k + 1 for k in evens))
        else:
            assert res["split"] is False
