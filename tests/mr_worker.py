"""One rank of a multi-rank engine run on a shared GPU (host-callback group
over gloo; see paper_2009_09523_b200/hostcomm.py).  Driven by
tests/test_multirank_gpu.py:  python mr_worker.py SCENARIO OUT.npz
with RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT in the environment
(WORLD_SIZE=1: no group, the single-process reference trajectory)."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_lib  # noqa: E402  (test infrastructure: data and init only)

SCEN = {
    # widths, act, loss, B, V, steps, mode
    "wide": ([128, 256, 256, 10], "relu", "softmax-cross-entropy", 96, 12, 4, "auto"),
    "node": ([784, 16, 10], "tanh", "softmax-cross-entropy", 96, 12, 4, "auto"),
    "ffma": ([64, 96, 48, 10], "relu", "softmax-cross-entropy", 96, 12, 4, "ffma"),
}


RESIZES = {2: ["gpu0", "gpu1"], 4: ["gpu0", "gpu1", "gpu5"]}   # step -> device ids


def trainer_run(model, rank, world, out):
    """The C++ drop-in Trainer (vnt_trainer C-ABI) on every process: 4 devices,
    resized to 2 (with 3 processes one goes idle) and then to 3 with a new id."""
    import paper_2009_09523_b200 as vnt
    comm = None
    if world > 1:
        from paper_2009_09523_b200 import hostcomm
        comm = hostcomm.world_group()
    widths, act, loss, B, V, steps, mode = SCEN[model]
    t = vnt.Trainer(widths, act, loss, 3, B, V, 0.05, 7, 4096, [(f"gpu{i}", 1 << 20) for i in range(4)],
                    gemm_mode=mode, comm=comm)
    losses = []
    for s in range(6):
        if s in RESIZES:
            t.resize([(d, 1 << 20) for d in RESIZES[s]])
        losses.append(t.step())
    params = t.params()
    stats = {}
    for i in range(t.local_device_count()):
        stats[i] = t.input_stats(i)
    np.savez(out, losses=np.array(losses), params=params,
             counts=np.array([stats[i][0] for i in sorted(stats)]),
             means=np.array([stats[i][1] for i in sorted(stats)]) if stats else np.zeros((0, widths[0])),
             m2s=np.array([stats[i][2] for i in sorted(stats)]) if stats else np.zeros((0, widths[0])),
             log=np.array([]))
    t.close()


def main():
    scenario, out = sys.argv[1], sys.argv[2]
    kind, _, model = scenario.partition(":")
    if kind == "trainer":
        rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("gloo", rank=rank, world_size=world)
        trainer_run(model, rank, world, out)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    import paper_2009_09523_b200 as vnt
    comm = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2009_09523_b200 import hostcomm
        comm = hostcomm.world_group()
    widths, act, loss, B, V, steps, mode = SCEN[model]
    port = oracle_lib.port()
    e = vnt.Engine(widths, act, loss, gemm_mode=mode, comm=comm,
                   momentum=0.5 if kind == "momentum" else 0.0)
    e.add_device(1 << 20)
    e.set_params(port.init_params(widths, 3))
    sizes = np.full(V, B // V, np.uint64)
    losses, logs = [], []

    def mapping(members):
        # node n -> the (n mod |members|)-th member; -1 elsewhere
        m = np.array([0 if members[n % len(members)] == rank else -1 for n in range(V)], np.int32)
        return m

    for s in range(steps if kind != "membership" else 6):
        x, y = port.synth_batch(7, 4096, widths[0], widths[-1], s * B, B)
        if kind in ("train", "momentum"):
            members = list(range(world))
            lo, _ = e.train_step(x, y, sizes, mapping(members), 0.05)
        elif kind == "membership":
            # steps 0-1 on every process, 2-3 on the first two (the others idle),
            # 4-5 on every process again (resize 3 -> 2 -> 3 without restart)
            if world > 1 and s in (2, 4):
                keep = s == 4 or rank < 2
                e.set_membership(keep, 0)
            members = list(range(world)) if (s < 2 or s >= 4) else list(range(min(2, world)))
            if rank not in members:
                losses.append(float("nan"))
                continue
            lo, _ = e.train_step(x, y, sizes, mapping(members), 0.05)
        elif kind == "decomposed":
            # reference decomposition: device_step on this rank's nodes (the last
            # rank has none), sync_gradients, sgd_apply
            mine = [n for n in range(V) if world == 1 or (n % max(1, world - 1) == rank and rank < world - 1)]
            if mine:
                off = np.cumsum([0] + [int(v) for v in sizes])
                xs = np.concatenate([x[off[n]:off[n + 1]] for n in mine])
                ys = np.concatenate([y[off[n]:off[n + 1]] for n in mine])
                e.device_step(0, xs, ys, sizes[mine])
            _, ls, ex = e.sync(want_grad=False)
            e.sgd_apply(0.05)
            lo = ls / ex
        else:
            raise SystemExit(f"unknown scenario {scenario}")
        losses.append(lo)
        logs.append(e.comm_log())
    params = e.get_params()
    np.savez(out, losses=np.array(losses), params=params,
             log=np.array([repr(l) for l in logs]))
    e.close()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
