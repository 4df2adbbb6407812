"""`vnt_train train` — the reference CLI's train command (tools/vnt.cpp:52-152)
on the drop-in Trainer: config strictness and exit codes (CPU), and on the GPU
the fig1 fixture against the reference's own outputs, byte-identical reruns,
1-device vs 4-device --compare-against divergence 0 (test_cli.cpp:58-137)."""
import json
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = Path(__file__).resolve().parent / "golden"


def _bin():
    p = ROOT / "build" / "bin" / "vnt_train"
    if not p.exists():
        from paper_2009_09523_b200 import build as b
        b.build_host()
        b.build_tools()
    if not p.exists():
        pytest.skip("vnt_train not built (nlohmann/json.hpp missing)")
    return p


def fig1_config(tmp, devices=4, **extra):
    g = json.loads((GOLDEN / "fig1_reference.json").read_text())["config"]
    cfg = {
        "workload": {"layer_widths": g["layer_widths"], "activation": g["activation"],
                     "loss": g["loss"], "seed": g["seed"]},
        "global_batch": g["global_batch"], "virtual_nodes": g["virtual_nodes"],
        "steps": g["steps"], "lr": g["lr"], "data_seed": g["data_seed"],
        "dataset_size": g["dataset_size"],
        "devices": [{"device_id": f"gpu{i}", "device_type": "B200", "memory_capacity": 256}
                    for i in range(devices)],
        "metrics_out": str(tmp / "metrics.jsonl"), "params_out": str(tmp / "params.json"),
    }
    cfg.update(extra)
    p = tmp / "cfg.json"
    p.write_text(json.dumps(cfg))
    return p


def run(*args):
    return subprocess.run([str(_bin()), *map(str, args)], capture_output=True, text=True,
                          timeout=300)


def test_usage_and_config_errors(tmp_path):
    assert run().returncode == 2
    bad = json.loads(fig1_config(tmp_path).read_text())
    bad["bogus"] = 1
    (tmp_path / "bad.json").write_text(json.dumps(bad))
    r = run("train", "--config", tmp_path / "bad.json")
    assert r.returncode == 2 and "unknown key" in r.stderr
    cap = json.loads(fig1_config(tmp_path).read_text())
    cap["virtual_nodes"] = 1                      # micro-batch 16 > capacity 8
    for d in cap["devices"]:
        d["memory_capacity"] = 8
    cap["devices"] = cap["devices"][:1]
    (tmp_path / "cap.json").write_text(json.dumps(cap))
    r = run("train", "--config", tmp_path / "cap.json")
    assert r.returncode == 3 and "gpu0" in r.stderr
    assert run("train", "--config", tmp_path / "missing.json").returncode == 2


@pytest.mark.gpu
def test_fig1_against_reference_outputs(tmp_path):
    g = json.loads((GOLDEN / "fig1_reference.json").read_text())
    r = run("train", "--config", fig1_config(tmp_path), "--json")
    assert r.returncode == 0, r.stderr
    summary = json.loads(r.stdout)
    assert summary["steps"] == 50 and summary["devices"] == 4
    lines = [json.loads(l) for l in (tmp_path / "metrics.jsonl").read_text().splitlines()]
    losses = np.array([l["loss"] for l in lines])
    want = np.array(g["step_losses"])
    assert np.max(np.abs(losses - want) / want) < 1e-5
    assert lines[0]["per_device"][0] == {"buffer_bytes": 1184, "device_id": "gpu0", "examples": 4,
                                         "peak_resident": 1, "waves": 4}
    params = json.loads((tmp_path / "params.json").read_text())
    assert [e["name"] for e in params["layout"]] == [n for n, _ in g["layout"]]
    assert np.abs(np.array(params["values"]) - np.array(g["final_params"])).max() < 1e-5
    # --compare-against the reference's checked-in params: within fp32 tolerance ...
    ref_params = tmp_path / "ref_params.json"
    ref_params.write_text(json.dumps({"layout": params["layout"], "values": g["final_params"]}))
    cfg = fig1_config(tmp_path, compare_tolerance=1e-5)
    r = run("train", "--config", cfg, "--compare-against", ref_params, "--json")
    assert r.returncode == 0, r.stderr
    assert 0 < json.loads(r.stdout)["max_divergence"] < 1e-5
    # ... and exit 4 at tolerance 0 (vnt.cpp:135-139)
    r = run("train", "--config", fig1_config(tmp_path), "--compare-against", ref_params)
    assert r.returncode == 4


@pytest.mark.gpu
def test_rerun_bytes_and_mapping_invariance(tmp_path):
    a, b, c = tmp_path / "a", tmp_path / "b", tmp_path / "c"
    for d in (a, b, c):
        d.mkdir()
    assert run("train", "--config", fig1_config(a, devices=4)).returncode == 0
    assert run("train", "--config", fig1_config(b, devices=4)).returncode == 0
    assert (a / "metrics.jsonl").read_bytes() == (b / "metrics.jsonl").read_bytes()
    assert (a / "params.json").read_bytes() == (b / "params.json").read_bytes()
    r = run("train", "--config", fig1_config(c, devices=1), "--compare-against", a / "params.json",
            "--json")
    assert r.returncode == 0, r.stderr
    s = json.loads(r.stdout)
    assert s["max_divergence"] == 0.0 and s["bitwise_identical"] is True


def test_profile_and_solve_commands(tmp_path, ref):
    """`vnt profile` / `vnt solve` (tools/vnt.cpp:154-263): curves from the cost
    model over the candidate grid, then the heterogeneous assignment — the same
    assignment the reference's own solver (oracle/_ref) finds on those curves."""
    wl = {"layer_widths": [4, 8, 2], "activation": "tanh", "loss": "mse", "seed": 1}
    models = [{"device_type": "V100", "fixed_overhead_s": 0.002, "per_example_cost_s": 0.00025,
               "comm_s": 0.01, "memory_capacity": 3072},
              {"device_type": "P100", "fixed_overhead_s": 0.002, "per_example_cost_s": 0.001,
               "comm_s": 0.01, "memory_capacity": 3072}]
    pcfg = tmp_path / "profile.json"
    pcfg.write_text(json.dumps({"workload": wl, "max_batch": 4096, "device_models": models,
                                "out_dir": str(tmp_path / "curves")}))
    r = run("profile", "--config", pcfg, "--json")
    assert r.returncode == 0, r.stderr
    paths = json.loads(r.stdout)["profiles"]
    curves = [json.loads(Path(p).read_text()) for p in paths]
    for m, c in zip(models, curves):
        # 2-device minus 1-device mean (reference semantics), so only up to rounding
        assert c["device_type"] == m["device_type"] and abs(c["comm_overhead_s"] - m["comm_s"]) < 1e-15
        for pt in c["points"]:   # mean of identical simulated times is that time, exactly
            assert pt["step_time_s"] == m["fixed_overhead_s"] + m["per_example_cost_s"] * pt["batch_size"]
        assert max(pt["batch_size"] for pt in c["points"]) <= m["memory_capacity"]
    scfg = tmp_path / "solve.json"
    scfg.write_text(json.dumps({"profiles": paths, "global_batch": 8192,
                                "pool": {"V100": {"count": 2, "memory_capacity": 3072},
                                         "P100": {"count": 2, "memory_capacity": 3072}},
                                "out": str(tmp_path / "plan" / "assignment.json")}))
    r = run("solve", "--config", scfg, "--json", "--explain")
    assert r.returncode == 0, r.stderr
    out = json.loads(r.stdout)
    a = out["assignment"]
    assert a == json.loads((tmp_path / "plan" / "assignment.json").read_text())
    got = {t["device_type"]: (t["count"], t["per_device_batch"], t["virtual_nodes"]) for t in a["types"]}
    assert got["V100"][1] == 3072 and got["P100"][1] == 1024          # test_hetero.cpp:107-134
    if ref is not None:
        import ctypes as C
        from test_hetero import _solve
        types = [dict(name=c["device_type"], count=2, cap=3072, comm=c["comm_overhead_s"],
                      points=[(p["batch_size"], p["step_time_s"]) for p in c["points"]])
                 for c in sorted(curves, key=lambda c: c["device_type"])]
        rc, res = _solve(ref.lib.vntref_hetero_solve, types, 8192)
        assert rc == 0
        best, t, cand = res
        assert t == a["predicted_step_time_s"] and cand == len(out["candidates"])
        assert {n: (k, b, v) for n, k, b, v in best} == got
    # infeasible -> exit 5 (vnt.cpp:395-413)
    scfg.write_text(json.dumps({"profiles": paths, "global_batch": 100000,
                                "pool": {"V100": {"count": 1, "memory_capacity": 64}}}))
    r = run("solve", "--config", scfg)
    assert r.returncode == 5 and "capacity" in r.stderr


@pytest.mark.gpu
def test_profile_measured_on_b200(tmp_path):
    """Extension key "measure": true — the curve is timed on this B200
    (hetero::profile_device) and feeds `vnt solve` like a synthetic one."""
    wl = {"layer_widths": [784, 16, 10], "activation": "tanh", "loss": "softmax-cross-entropy",
          "seed": 11}
    pcfg = tmp_path / "profile.json"
    pcfg.write_text(json.dumps({"workload": wl, "max_batch": 64, "steps": 20, "out_dir": str(tmp_path),
                                "device_models": [{"device_type": "B200", "fixed_overhead_s": 0.0,
                                                   "per_example_cost_s": 1e-6, "comm_s": 0.0,
                                                   "memory_capacity": 64, "measure": True}]}))
    r = run("profile", "--config", pcfg, "--json")
    assert r.returncode == 0, r.stderr
    c = json.loads((tmp_path / "B200.json").read_text())
    assert [p["batch_size"] for p in c["points"]] == [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64]
    assert all(0 < p["step_time_s"] < 0.05 for p in c["points"])
    scfg = tmp_path / "solve.json"
    scfg.write_text(json.dumps({"profiles": [str(tmp_path / "B200.json")], "global_batch": 256,
                                "pool": {"B200": {"count": 8, "memory_capacity": 64}}}))
    r = run("solve", "--config", scfg, "--json")
    assert r.returncode == 0, r.stderr
    (t,) = json.loads(r.stdout)["assignment"]["types"]
    assert t["count"] * t["per_device_batch"] == 256
