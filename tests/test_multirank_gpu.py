"""The engine's multi-rank paths with several processes on ONE GPU.

Each rank is a separate process with its own engine on cuda:0; the process
group is a host-callback group over gloo (vnt_comm_ops, hostcomm.py), so the
ranks exchange through the host and no kernel waits on another rank's.  This
runs the real engine code of an N-GPU step — node n on rank n mod N, the
sharded update (per-layer reduce-scatter, 1/N update, weight all-gather), the
all-reduce path, the reference decomposition with a rank that hosts no node,
and an elastic resize 3 -> 2 -> 3 by pool membership — and checks the
north-star claim: the trajectory is bit-identical to one process for a fixed V.
"""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def launch(scenario, world, tmp_path, extra_env=None):
    port = _port()
    procs, outs = [], []
    for r in range(world):
        out = tmp_path / f"{scenario.replace(':', '_')}_{world}_{r}.npz"
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), **(extra_env or {}))
        procs.append(subprocess.Popen([sys.executable, str(HERE / "mr_worker.py"), scenario, str(out)],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                      text=True))
        outs.append(out)
    logs = []
    for p in procs:
        try:
            o, _ = p.communicate(timeout=600)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        logs.append(o)
        assert p.returncode == 0, o[-4000:]
    return [np.load(o) for o in outs]


@pytest.mark.parametrize("scenario,world,shard", [("train:wide", 2, "1"), ("train:wide", 3, "1"),
                                                  ("train:wide", 2, "0"), ("train:node", 2, "1"),
                                                  ("train:ffma", 3, "1"),
                                                  ("momentum:wide", 2, "1")])
def test_ranks_match_single_process_bitwise(tmp_path, scenario, world, shard):
    ref = launch(scenario, 1, tmp_path)[0]
    got = launch(scenario, world, tmp_path, {"VNT_SHARD": shard})
    for r, g in enumerate(got):
        assert np.array_equal(g["losses"], ref["losses"]), (r, g["losses"], ref["losses"])
        assert np.array_equal(g["params"], ref["params"]), r
    # every rank issued the identical collective sequence
    for g in got[1:]:
        assert list(g["log"]) == list(got[0]["log"])


def test_decomposed_path_with_an_idle_rank(tmp_path):
    """device_step / sync_gradients / sgd_apply with a rank that hosts no node
    (it joins the first-round scale agreement from sync: ADVICE r1)."""
    ref = launch("decomposed:wide", 1, tmp_path)[0]
    got = launch("decomposed:wide", 3, tmp_path)
    for g in got:
        assert np.array_equal(g["params"], ref["params"])
        assert np.allclose(g["losses"], ref["losses"], rtol=0, atol=1e-12)


def test_resize_by_pool_membership(tmp_path):
    """3 processes -> 2 (the third idles, no restart) -> 3 again; the
    training trajectory equals one process throughout (cfg5 shape)."""
    ref = launch("membership:wide", 1, tmp_path)[0]
    got = launch("membership:wide", 3, tmp_path)
    for r, g in enumerate(got):
        assert np.array_equal(g["params"], ref["params"]), r
        mask = ~np.isnan(g["losses"])
        assert np.array_equal(g["losses"][mask], ref["losses"][mask]), r


@pytest.mark.parametrize("world", [2, 3])
def test_trainer_processes_with_resize(tmp_path, world):
    """The C++ drop-in Trainer with one process per rank (round-robin device
    placement) through resizes 4 -> 2 -> 3 devices (a new id; with 3
    processes one idles and rejoins): parameters and every device's input
    statistics bitwise equal to the single-process Trainer's."""
    ref = launch("trainer:wide", 1, tmp_path)[0]
    got = launch("trainer:wide", world, tmp_path)
    final = ["gpu0", "gpu1", "gpu5"]                 # ascending ids after the last resize
    placed = {"gpu0": 0, "gpu1": 1, "gpu2": 2 % world, "gpu3": 3 % world, "gpu5": 4 % world}
    for r, g in enumerate(got):
        mine = [final.index(d) for d in final if placed[d] == r]
        mask = ~np.isnan(g["losses"])
        assert np.array_equal(g["losses"][mask], ref["losses"][mask]), r
        if mine:   # trains at the end: holds the current replica
            assert mask[-1] and np.array_equal(g["params"], ref["params"]), r
        assert list(g["counts"]) == [ref["counts"][i] for i in mine], r
        for k, i in enumerate(mine):
            assert np.array_equal(g["means"][k], ref["means"][i]) and np.array_equal(g["m2s"][k], ref["m2s"][i])
