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
