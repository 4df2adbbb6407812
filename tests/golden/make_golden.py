"""Generate the committed golden fixtures in tests/golden/ (run in the dev
container, where /root/reference exists; the GPU box only reads the outputs).

1. fig1_reference.json — the reference's own checked-in outputs for
   fixtures/fig1_train.json (out/fig1_metrics.jsonl: 50 per-step losses;
   out/fig1_params.json: 148 final params), re-encoded as one JSON object.
2. ref_<name>.npz — trajectories produced by the reference itself
   (oracle/_ref/libvntref.so, built from /root/reference by oracle/Makefile):
   per-step losses, final params, and device-0 input statistics.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
import oracle_lib  # noqa: E402

REF_OUT = Path("/root/reference/proj/out")

# name: (widths, act, loss, seed, B, V, lr, data_seed, dataset_size, devices, steps)
CASES = {
    # acceptance.cpp:57-67 headline workload, 200 steps
    "headline": ([4, 16, 4], "tanh", "mse", 11, 64, 8, 0.05, 11, 256, 8, 200),
    # BASELINE config 1/2 shape ([784,16,10] tanh/CE, B=256, V=16), 20 steps
    "cfg1": ([784, 16, 10], "tanh", "softmax-cross-entropy", 11, 256, 16, 0.05, 11, 60000, 1, 20),
    # wide-MLP topology (cfg3) at reduced width so the fp64 exact oracle finishes in seconds
    "wide_small": ([784, 256, 256, 10], "relu", "softmax-cross-entropy", 1, 512, 8, 0.01, 1, 65536, 1, 4),
}


def fig1():
    losses = [json.loads(l)["loss"] for l in (REF_OUT / "fig1_metrics.jsonl").read_text().splitlines() if l.strip()]
    params = json.loads((REF_OUT / "fig1_params.json").read_text())
    out = {
        "config": {"layer_widths": [4, 16, 4], "activation": "tanh", "loss": "mse", "seed": 11,
                   "global_batch": 16, "virtual_nodes": 16, "steps": 50, "lr": 0.05,
                   "data_seed": 11, "dataset_size": 64, "devices": 4},
        "source": "reference proj/out/fig1_metrics.jsonl + proj/out/fig1_params.json",
        "step_losses": losses,
        "final_params": params["values"],
        "layout": [[e["name"], e["shape"]] for e in params["layout"]],
    }
    (HERE / "fig1_reference.json").write_text(json.dumps(out, indent=1))


def traj(name):
    widths, act, loss, seed, B, V, lr, ds, n, G, steps = CASES[name]
    r = oracle_lib.ref()
    assert r is not None, "build oracle/_ref first (make -C oracle ref)"
    t = r.trainer(widths, act, loss, seed, B, V, lr, ds, n, G)
    losses = np.array([t.step() for _ in range(steps)])
    cnt, mean, m2 = t.input_stats(0)
    np.savez_compressed(HERE / f"ref_{name}.npz", losses=losses, params=t.params(),
                        stats_count=np.array(cnt), stats_mean=mean, stats_m2=m2,
                        config=np.array(json.dumps(dict(zip(
                            ["widths", "act", "loss", "seed", "B", "V", "lr", "data_seed",
                             "dataset_size", "devices", "steps"], CASES[name])))))


if __name__ == "__main__":
    fig1()
    for k in CASES:
        traj(k)
    print("golden fixtures written to", HERE)
