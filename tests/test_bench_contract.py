"""bench.py's JSON-line contract on the CPU: the reference arm (the oracle, --impl reference) prints
one line with the driver's keys on rank 0 and nothing on other ranks; the expected-counts file the
GPU arm's parity gate reads is complete for every config.  (The GPU arm itself runs on the B200.)"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

REQUIRED = ["impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"]


def _run(env_extra, *args):
    env = dict(os.environ, **env_extra)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=env,
                          capture_output=True, text=True, timeout=600)


def test_reference_arm_line_rank0():
    r = _run({"RANK": "0"}, "--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "3")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in REQUIRED:
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["unit"] == "wedges/s" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_other_ranks_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2"}, "--impl", "reference", "--config", "1", "--gpus", "2")
    assert r.returncode == 0, r.stderr[-2000:]
    assert not [l for l in r.stdout.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("config", [1, 2, 3, 4, 5, 6])
def test_expected_counts_complete(config):
    with open(os.path.join(ROOT, "tests", "golden", "expected_counts.json")) as f:
        exp = json.load(f)
    e = exp[f"config{config}"]
    for k in ("graph_sha256", "B", "N", "W_G", "pv_sha256"):
        assert k in e, (config, k)
    assert e["B"] >= 0 and e["N"] >= 0 and e["W_G"] > 0
    assert len(e["graph_sha256"]) == 64 and len(e["pv_sha256"]) == 64
