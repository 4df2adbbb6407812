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
