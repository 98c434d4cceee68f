"""Host-side pieces of bench.py (no GPU): the roofline inputs it reads from profiles/, the metric name and the
workload description, and the reference arm's JSON contract on a tiny sample."""
import json
import os
import subprocess
import sys

import pytest

import fctgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_metric_is_baselines():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert json.load(f)["metric"] == bench.METRIC


def _capture(tmp_path, monkeypatch):
    cap = {"workload": {"config": 4, "n": fctgen.CONFIGS[4].n, "d": 64},
           "kernels": {"fct1_sketch": {"kernel": "void <unnamed>::sketch_v5_kernel<5, 5, 8, 2, 1>(CUtensorMap_st, ...)",
                                       "dram_bytes_read": 18.0e9, "dram_bytes_write": 5e6,
                                       "limiter": {"resource": "shared-memory data pipe", "pct_of_peak": 80.0}},
                       "l1_rownorm": {"kernel": "void <unnamed>::rownorm_ws2_kernel<27, 64, 3, 0, 1, 0>(...)",
                                      "dram_bytes_read": 17.3e9, "dram_bytes_write": 3.6e8}}}
    (tmp_path / "profiles").mkdir()
    (tmp_path / "profiles" / "cap.json").write_text(json.dumps(cap))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    monkeypatch.setattr(bench, "TRAFFIC_FILE", os.path.join("profiles", "cap.json"))


def test_traffic_only_for_the_captured_workload_and_kernel_instances(tmp_path, monkeypatch):
    _capture(tmp_path, monkeypatch)
    cfg = fctgen.CONFIGS[4]
    inst = {"fct1_sketch": "sketch_v5_kernel<5, 5, 8, 2, 1>", "l1_rownorm": "rownorm_ws2_kernel<27, 64, 3, 0, 1, 0>"}
    t = bench.load_traffic(cfg, cfg.n, 1, inst)
    assert t["fct1_sketch"] > 0 and t["l1_rownorm"] > 0 and "dram__bytes_read.sum" in t["_source"]
    assert t["_limiter"]["fct1_sketch"]["pct_of_peak"] == 80.0
    # another kernel instance than the captured one: no traffic claimed for it
    t2 = bench.load_traffic(cfg, cfg.n, 1, dict(inst, fct1_sketch="sketch_v1_kernel<5, 5, 8, 2, 1>"))
    assert "fct1_sketch" not in t2 and t2["_mismatch"]["fct1_sketch"]["launched"].startswith("sketch_v1")
    assert t2["l1_rownorm"] > 0
    # another shard size or world size is not the captured launch: no traffic claimed
    assert bench.load_traffic(cfg, cfg.n // 2, 2, inst) == {}
    assert bench.load_traffic(fctgen.CONFIGS[3], fctgen.CONFIGS[3].n, 1, inst) == {}


def test_peaks_have_a_source():
    peak, src = bench.load_peaks()
    assert peak > 1000 and isinstance(src, str) and src


def test_workload_description_names_the_config():
    cfg = fctgen.CONFIGS[4]
    w = bench.workload_desc(cfg, cfg.n)
    assert "cfg4" in w and str(cfg.n) in w and f"r1={cfg.r1}" in w


def test_reference_arm_json_line():
    """--impl reference (the oracle on the host cores) prints one JSON line with the contract's keys."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "1", "--cpu-blocks", "2"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "config",
              "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0 and line["warmup"] >= 3
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "oracle"
